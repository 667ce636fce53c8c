#!/bin/bash
# ncu launch list (gpu__time_duration per kernel) of a short bench run.
TAG=${1:-r01}; W=${2:-cfg3}; shift 2
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/${TAG}_launches_bench.txt 2>&1
tail -1 gpurun_out/${TAG}_launches_bench.txt | cut -c1-200
