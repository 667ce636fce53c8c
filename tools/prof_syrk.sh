#!/bin/bash
# SYRK kernel evidence: A/B timings of the debug-skip variants (profiling
# only: results invalid) and one ncu --set full capture (with source) of an
# unranged cfg3 SYRK launch. Usage: tools/prof_syrk.sh TAG [workload]
TAG=${1:-r02}; W=${2:-cfg3}
mkdir -p gpurun_out
for v in "" "E3_DEBUG_SKIP=1" "E3_DEBUG_SKIP=2" "E3_DEBUG_SKIP=3" "E3_DEBUG_SKIP=4"; do
  env $v timeout 300 python tools/syrk_time.py --workload $W --tag "$TAG:$v" 2>&1 | tail -1
done | tee gpurun_out/${TAG}_skip_${W}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_syrk_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_search_${W} -f \
    python tools/syrk_time.py --workload $W --lo 0.25 --hi 0.26 --reps 1 > gpurun_out/${TAG}_ncu_${W}.txt 2>&1
tail -3 gpurun_out/${TAG}_ncu_${W}.txt
