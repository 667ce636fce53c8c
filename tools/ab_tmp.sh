for rep in 1 2; do
timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/o.json 2> /tmp/o.err; echo "ring+fence rc=$? $(python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print(round(d['value'],1))")"
E3_NO_YRING=1 timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e > /tmp/o.json 2> /tmp/o.err; echo "noring rc=$? $(python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print(round(d['value'],1))")"
done
