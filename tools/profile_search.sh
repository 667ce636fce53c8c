#!/bin/bash
# One ncu --set full capture of an (unranged) SYRK search launch at cfg3.
TAG=${1:-r01b}; W=${2:-cfg3}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:search_syrk -s 5 -c 1 \
    -o gpurun_out/${TAG}_search_${W} -f \
    python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_full.txt 2>&1
tail -2 gpurun_out/${TAG}_ncu_full.txt
