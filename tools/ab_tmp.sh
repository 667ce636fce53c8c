E3_LIBCU=build/v_e16/libepi3cu.so timeout 1200 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for W in cfg3 cfg5 cfg2; do
for n in cur10 e16; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
