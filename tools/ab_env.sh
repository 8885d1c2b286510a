#!/bin/bash
# A/B of plan knobs: tools/ab_env.sh CONFIG "ENV1" "ENV2" ... -> one bench line per setting
# (kernels_ms + value) into gpurun_out/ab_cfgCONFIG.txt
cfg=$1; shift
out=gpurun_out/ab_cfg${cfg}.txt
for e in "$@"; do
  echo "== $e" >> $out
  env $e python bench.py --config $cfg --no-cpu-baseline --steps 300 --warmup 10 2>>$out | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value'],1), d['e2e']['value'] and round(d['e2e']['value'],1), {k: round(v*1e3,2) for k,v in d['kernels_ms'].items()}, d['clocks']['sm_mhz'], d.get('schedule'))" >> $out 2>&1
done
