#!/bin/bash
# Round-end ncu evidence in one gpurun call (each ncu pass after its own command exited 0 without ncu):
#  config 4: launch list of bench.py in the timed (mid-solve) window; --set full of support_a in the dense phase
#  config 3: launch list + --set full of the slab sweep; config 2: launch list
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_ncu_final.sh TAG'
TAG=${1:-r02s5}
O=gpurun_out; mkdir -p $O
ITER='regex:gemv|hemv|zupdate|support|finalize|sweep|objective|rows'
B4="python bench.py --config 4 --steps 30 --warmup 5 --no-cpu-baseline"
$B4 > $O/${TAG}_plain4.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -k "$ITER" -s 4100 -c 80 --csv \
    --log-file $O/${TAG}_cfg4_launches.csv $B4 > $O/${TAG}_ncul4.log 2>&1
echo "cfg4 launch list exit $?"
P4="python tools/profile_step.py --config 4 --iters 10"
$P4 > $O/${TAG}_plainp4.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:support_a" -s 7 -c 1 -f \
    -o $O/${TAG}_cfg4_support_a $P4 > $O/${TAG}_ncup4.log 2>&1
echo "cfg4 support_a capture exit $?"
for c in 3 2; do
  B="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline"
  $B > $O/${TAG}_plain$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -k "$ITER" -c 300 --csv \
      --log-file $O/${TAG}_cfg${c}_launches.csv $B > $O/${TAG}_ncul$c.log 2>&1
  echo "cfg$c launch list exit $?"
done
P3="python tools/profile_step.py --config 3 --iters 3"
$P3 > $O/${TAG}_plainp3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:sweep_slab" -s 2 -c 1 -f \
    -o $O/${TAG}_cfg3_sweep_slab $P3 > $O/${TAG}_ncup3.log 2>&1
echo "cfg3 sweep capture exit $?"
ls -la $O/${TAG}_*
