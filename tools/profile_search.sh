#!/bin/bash
# One ncu --set full capture of the search kernel (cfg3, 1/1024 slice).
TAG=${1:-r01b}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:search_syrk -s 1 -c 1 \
    -o gpurun_out/${TAG}_search_cfg3 -f \
    python bench.py --workload cfg3 --steps 1 --warmup 1 --slices 1024 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_full.txt 2>&1
tail -2 gpurun_out/${TAG}_ncu_full.txt
