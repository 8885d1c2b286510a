#!/bin/bash
# One gpurun call: ncu launch list of the bench command + one --set full capture of the top kernel.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_ncu.sh TAG CONFIG KERNEL_REGEX'
TAG=${1:-r02}; CFG=${2:-4}; KRE=${3:-gemv_h}
O=gpurun_out; mkdir -p $O
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline"
ITER='regex:gemv|hemv|zupdate|support|finalize|sweep|objective|rows'
$CMD > $O/${TAG}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -k "$ITER" -c 300 --csv \
    --log-file $O/${TAG}_cfg${CFG}_launches.csv $CMD > $O/${TAG}_ncu1.log 2>&1
echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 2 -c 2 -f \
    -o $O/${TAG}_cfg${CFG}_${KRE} python tools/profile_step.py --config $CFG --iters 3 > $O/${TAG}_ncu2.log 2>&1
echo "full capture exit $?"
tail -3 $O/${TAG}_ncu1.log $O/${TAG}_ncu2.log
