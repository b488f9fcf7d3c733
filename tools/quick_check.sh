python -m pytest tests -m gpu -x -q > gpurun_out/tq.log 2>&1; tail -2 gpurun_out/tq.log
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bq.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1]);print('value',d['value'],'step',d['ms_per_step'],'e2e',d['e2e']['value'],d['kernels_ms'],'ga',d['ga']['ms_per_generation'])"
