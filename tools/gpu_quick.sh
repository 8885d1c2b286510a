#!/bin/bash
# GPU tests + the three single-scene bench lines, no CPU baseline. usage: bash tools/gpu_quick.sh TAG [pytest args]
TAG=${1:-q}; shift
O=gpurun_out; mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -x -q "$@" ) > $O/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest.log
for c in 4 2 3; do python bench.py --config $c --no-cpu-baseline > $O/${TAG}_bench_cfg$c.json 2> $O/${TAG}_bench_cfg$c.err; done
tail -4 $O/${TAG}_pytest.log
python - <<PY
import json
for c in (4,2,3):
    try:
        d=json.loads(open('$O/${TAG}_bench_cfg%d.json'%c).read().strip().splitlines()[-1])
        print(c, round(d['value'],1),'it/s e2e',round(d['e2e']['value'],1),'setup',round(d['run']['setup_s'],3), d['clocks']['sm_mhz'])
    except Exception as e: print(c,'ERR',e)
PY
