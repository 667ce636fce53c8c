timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
E3_LIBCU=build/v_tl7/libepi3cu.so timeout 300 python tools/syrk_time.py --workload cfg4 --lo 0.25 --hi 0.27 --reps 1 > gpurun_out/tl_cfg4c.txt 2>&1
