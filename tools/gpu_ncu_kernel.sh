#!/bin/bash
# One --set full capture of a kernel of tools/profile_step.py (after a plain run of the same command).
# usage: bash tools/gpu_ncu_kernel.sh TAG CONFIG KERNEL_REGEX [SKIP] [COUNT]
TAG=$1; CFG=$2; KRE=$3; SKIP=${4:-0}; CNT=${5:-1}
O=gpurun_out; mkdir -p $O
CMD="python tools/profile_step.py --config $CFG --iters 3"
$CMD > $O/${TAG}_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s $SKIP -c $CNT -f \
    -o $O/${TAG}_cfg${CFG}_${KRE} $CMD > $O/${TAG}_ncu.log 2>&1
echo "capture exit $?"; tail -n 3 $O/${TAG}_ncu.log
