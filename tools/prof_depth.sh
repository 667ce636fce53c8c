# stage-depth sensitivity: default (smem scratch, 2 stages) vs global scratch with 3 / 2 stages,
# full scoring and E3_DEBUG_SKIP=1 (pipeline-bound); profiling build
P=build/v_prof/libepi3cu.so
for v in "" "E3_NO_SMEM_SCRATCH=1" "E3_NO_SMEM_SCRATCH=1 E3_SYRK_STAGES=2" "E3_DEBUG_SKIP=1" "E3_DEBUG_SKIP=1 E3_NO_SMEM_SCRATCH=1" "E3_DEBUG_SKIP=1 E3_NO_SMEM_SCRATCH=1 E3_SYRK_STAGES=2" "E3_DEBUG_SKIP=3 E3_NO_SMEM_SCRATCH=1"; do
  env E3_LIBCU=$P $v timeout 300 python tools/syrk_time.py --workload cfg3 --tag "$v" 2>&1 | tail -1
done | tee gpurun_out/depth_cfg3.txt
