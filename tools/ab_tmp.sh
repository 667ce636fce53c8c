E3_LIBCU=build/v_pd4/libepi3cu.so timeout 300 python -m pytest tests/test_gpu_bench_path.py -x -q -m gpu 2>&1 | tail -1
for W in cfg4 cfg5 cfg3 cfg2; do
for n in pd3 pd4; do W=$W timeout 300 bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
