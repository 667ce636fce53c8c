#!/bin/bash
# End-of-session evidence in one GPU call: tests, smoke, the driver's bench
# commands (both arms), the other configs, a launch list and ncu --set full
# captures of the SYRK search kernel and the pair-index kernel. TAG names the set.
TAG=${1:-r02d}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -5 | tee gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_cfg3_driver_cmd.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_reference_driver_cmd.json 2>> gpurun_out/${TAG}_bench.err; echo "ref rc=$?"
for W in cfg2 cfg4 cfg5; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 2>>gpurun_out/${TAG}_bench.err | tail -1 > gpurun_out/${TAG}_bench_${W}.json
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_launches_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_syrk_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_search_cfg3 -f python tools/syrk_time.py --workload cfg3 --lo 0.25 --hi 0.26 --reps 1 > gpurun_out/${TAG}_ncu_search.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pairs_tc -c 1 \
    -o gpurun_out/${TAG}_pairs_cfg3 -f python tools/syrk_time.py --workload cfg3 --lo 0.25 --hi 0.2501 --reps 1 > gpurun_out/${TAG}_ncu_pairs.txt 2>&1
ls gpurun_out | grep $TAG
