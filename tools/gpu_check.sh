#!/bin/bash
# One GPU round: smoke, parity tests, a short bench and the ncu launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 | tee gpurun_out/smoke.txt
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --workload cfg2 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -3 | tee gpurun_out/bench_cfg2.txt
timeout 900 python bench.py --steps 3 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench_cfg3.txt
