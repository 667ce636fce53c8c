timeout 900 python tools/repeat_create_check.py cfg2 60 2>&1 | tail -2
timeout 900 python tools/repeat_create_check.py cfg2 20 tc_masked 2>&1 | tail -2
timeout 900 python tools/repeat_create_check.py cfg1 100 2>&1 | tail -2
timeout 900 python tools/repeat_create_check.py cfg4 15 2>&1 | tail -2
