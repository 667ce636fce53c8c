# A/B: correctness (bench-path + parity subsets) on the in-tree build, then timings of
# build/v_<name> variants vs the in-tree build on cfg3 / cfg5 / cfg2.  usage: ab_run.sh name...
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bench_path.py -x -q -m gpu 2>&1 | tail -2
for W in ${WS:-cfg3 cfg5 cfg2}; do
  for n in "$@"; do
    W=$W ARGS="${ARGS:-}" bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"
  done
  W=$W ARGS="${ARGS:-}" bash tools/ab_syrk.sh "tree=paper_2201_10956_b200/libepi3cu.so"
done
