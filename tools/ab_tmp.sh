timeout 600 python tools/repeat_check.py cfg3 30 2>&1 | tail -2
timeout 600 python tools/repeat_check.py cfg5 100 2>&1 | tail -2
timeout 600 python tools/repeat_check.py cfg2 300 2>&1 | tail -2
