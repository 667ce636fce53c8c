./tools/tmem_layout_probe 2>&1 | tee gpurun_out/tmem_probe.txt
timeout 1200 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for W in cfg4 cfg3; do
for n in base9 cur9; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
