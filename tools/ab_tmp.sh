E3_LIBCU=build/v_md/libepi3cu.so timeout 1200 python -m pytest tests/test_gpu_bench_path.py -x -q -m gpu 2>&1 | tail -1
E3_LIBCU=build/v_mdtl/libepi3cu.so python tools/syrk_time.py --workload cfg3 --lo 0.25 --hi 0.253 --reps 1 > gpurun_out/mdtl2.txt 2>&1
for W in cfg3 cfg5 cfg2; do
for n in cur11 md; do W=$W bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
