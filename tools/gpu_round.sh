#!/bin/bash
# One GPU call: new bench-path tests, sanitizer, smoke, the full -m gpu suite,
# then the driver's exact bench commands (both arms). Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 600 python -m pytest tests/test_gpu_bench_path.py -x -q -m gpu 2>&1 | tail -30 | tee gpurun_out/pytest_bench_path.txt
E3_SYRK_YBUDGET_KIB=16 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_multibatch.py 2>&1 | tail -15 | tee gpurun_out/sanitize.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 | tee gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver.json 2> gpurun_out/bench_driver.err; echo "bench rc=$?" | tee -a gpurun_out/bench_driver.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?" | tee -a gpurun_out/bench_reference.err
