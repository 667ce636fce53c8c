for rep in 1 2; do
for n in d3all dmode; do
E3_LIBCU=build/v_$n/libepi3cu.so timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['value'],2))"
done; done
