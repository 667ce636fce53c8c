timeout 900 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for W in cfg3 cfg5 cfg2; do
for n in mma2; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
W=$W bash tools/ab_syrk.sh "tree=paper_2201_10956_b200/libepi3cu.so"
done
