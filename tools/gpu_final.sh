#!/bin/bash
# The driver's round-end sequence in one gpurun call: GPU tests, smoke(), both bench arms with its arguments.
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_final.sh TAG'
TAG=${1:-final}
O=gpurun_out; mkdir -p $O
( time timeout 2400 python -m pytest tests -x -q -m gpu ) > $O/${TAG}_pytest.log 2>&1
grep -n "passed\|failed" $O/${TAG}_pytest.log | tail -2
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; tail -1 $O/${TAG}_smoke.log
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
tail -4 $O/${TAG}_bench.err
python - <<PY
import json
r=json.loads(open('$O/${TAG}_bench_reference.json').read().strip().splitlines()[-1])
d=json.loads(open('$O/${TAG}_bench.json').read().strip().splitlines()[-1])
print('reference', r['value'], r['ms_per_step'], r['cpu_baseline']['cores'])
print('ours', round(d['value'],2), d['ms_per_step'], 'e2e', round(d['e2e']['value'],2), 'whole', round(d['run']['whole_solve']['iterations_per_s'],2), d['roofline']['frac'], d['clocks'], d['gpu_launches'], 'same_config', r['config']==d['config'])
print('cpu_baseline', d.get('cpu_baseline',{}).get('value'))
PY
