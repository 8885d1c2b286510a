#!/bin/bash
# ncu captures of the sweep on configs 2 and 3 + their launch lists (one gpurun call).
TAG=${1:-r02}; O=gpurun_out; mkdir -p $O
for c in 3 2; do
  CMD="python tools/profile_step.py --config $c --iters 3"
  $CMD > $O/${TAG}_plain_cfg$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:sweep_slab -s 2 -c 1 -f -o $O/${TAG}_cfg${c}_sweep_slab $CMD > $O/${TAG}_ncu_cfg$c.log 2>&1
  echo "cfg $c capture exit $?"
  BCMD="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline"
  $BCMD > $O/${TAG}_plainb_cfg$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:gemv|hemv|zupdate|support|finalize|sweep|objective|rows' -c 200 --csv --log-file $O/${TAG}_cfg${c}_launches.csv $BCMD > $O/${TAG}_ncul_cfg$c.log 2>&1
  echo "cfg $c launch list exit $?"
done
