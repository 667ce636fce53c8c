E3_LIBCU=build/v_ps4/libepi3cu.so timeout 1200 python -m pytest tests/test_gpu_bench_path.py -x -q -m gpu 2>&1 | tail -1
for W in cfg3 cfg5 cfg2 cfg4; do
for n in kb64 ps3 ps4; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
