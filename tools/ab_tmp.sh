timeout 900 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for W in cfg3 cfg5 cfg2; do
W=$W bash tools/ab_syrk.sh "cur3=build/v_cur3/libepi3cu.so"
W=$W bash tools/ab_syrk.sh "tree=paper_2201_10956_b200/libepi3cu.so"
done
