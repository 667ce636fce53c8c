timeout 1200 python -m pytest tests/test_gpu_bench_path.py -x -q -m gpu 2>&1 | tail -1
for W in cfg3 cfg5 cfg2 cfg4; do
W=$W bash tools/ab_syrk.sh "cur11=build/v_cur11/libepi3cu.so"
W=$W bash tools/ab_syrk.sh "tree=paper_2201_10956_b200/libepi3cu.so"
done
