#!/bin/bash
# ncu evidence for profiles/: the launch list of a bench run and one full
# capture of the search kernel (never a multi-rank command).
set -x
mkdir -p gpurun_out
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --workload cfg3 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_launches_bench.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 \
    -o gpurun_out/${TAG}_search_cfg3 -f \
    python bench.py --workload cfg3 --steps 1 --warmup 1 --slices 1024 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_full.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:pairs_kernel -c 1 \
    -o gpurun_out/${TAG}_pairs_cfg3 -f \
    python bench.py --workload cfg3 --steps 1 --warmup 0 --slices 4096 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out
