mkdir -p gpurun_out
P=build/v_prof/libepi3cu.so
for v in "" "E3_DEBUG_SKIP=1" "E3_DEBUG_SKIP=2" "E3_DEBUG_SKIP=3" "E3_DEBUG_SKIP=4" "E3_DEBUG_SKIP=5"; do
  env E3_LIBCU=$P $v timeout 300 python tools/syrk_time.py --workload cfg3 --tag "skip:$v" 2>&1 | tail -1
done | tee gpurun_out/p1_skip_cfg3.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_syrk_kernel -s 3 -c 1 \
    -o gpurun_out/p1_search_cfg3 -f \
    python tools/syrk_time.py --workload cfg3 --lo 0.25 --hi 0.26 --reps 1 > gpurun_out/p1_ncu.txt 2>&1
tail -3 gpurun_out/p1_ncu.txt
