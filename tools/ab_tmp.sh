E3_LIBCU=build/v_pair/libepi3cu.so timeout 300 python -m pytest tests/test_gpu_bench_path.py -x -q -m gpu 2>&1 | tail -1
E3_LIBCU=build/v_pairtl/libepi3cu.so timeout 300 python tools/syrk_time.py --workload cfg3 --lo 0.25 --hi 0.253 --reps 1 > gpurun_out/pairtl2.txt 2>&1
for W in cfg3 cfg5; do
for n in nopair pair; do W=$W timeout 300 bash tools/ab_syrk.sh "$n=build/v_$n/libepi3cu.so"; done
done
