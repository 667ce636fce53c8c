#!/bin/bash
# Evidence for profiles/: launch list of a cfg3 bench step, one ncu --set full
# capture each of the SYRK search kernel (unranged launch) and the pair-index
# kernel, a full bench line, and the engine/config sweep. One GPU, never
# multi-rank under ncu.
TAG=${1:-r01x}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_launches_bench.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:search_syrk -s 5 -c 1 \
    -o gpurun_out/${TAG}_search_cfg3 -f \
    python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_search.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:pairs_tc -c 1 \
    -o gpurun_out/${TAG}_pairs_cfg3 -f \
    python bench.py --workload cfg3 --steps 1 --warmup 0 --slices 4096 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_pairs.txt 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_cfg3.json 2> gpurun_out/${TAG}_bench_cfg3.err
for W in cfg2 cfg4 cfg5; do
  python bench.py --workload $W --steps 3 --warmup 3 --no-cpu 2>/dev/null | tail -1 > gpurun_out/${TAG}_bench_${W}.json
done
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1
ls -la gpurun_out | tail -20
