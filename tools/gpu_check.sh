#!/bin/bash
# One gpurun call: GPU tests, bench lines (ours + reference arm), ncu launch list.
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_check.sh TAG'
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${TAG}_smi.txt 2>&1
( time timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 ) > $O/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest.log
( time python bench.py ) > $O/${TAG}_bench_cfg4.json 2> $O/${TAG}_bench_cfg4.err
( time python bench.py --impl reference ) > $O/${TAG}_bench_cfg4_reference.json 2> $O/${TAG}_bench_cfg4_reference.err
python bench.py --config 2 --steps 600 > $O/${TAG}_bench_cfg2.json 2> $O/${TAG}_bench_cfg2.err
python bench.py --config 3 --steps 600 > $O/${TAG}_bench_cfg3.json 2> $O/${TAG}_bench_cfg3.err
tail -3 $O/${TAG}_pytest.log
cat $O/${TAG}_bench_cfg4.json | cut -c1-600
