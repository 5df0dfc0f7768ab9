#!/bin/bash
# ncu evidence for one hgemv configuration (1 GPU).
# usage: bash tools/gpu_prof.sh [cfg] [tag] [dense-kernel-regex] [coupling-regex] [coupling-skip]
CFG=${1:-cfg2}; TAG=${2:-r01}
KDENSE=${3:-seg_gemm_kernelILi64ELi32ELi4ELi1ELi3ELb1ELi2E}
KCOUP=${4:-seg_gemm_kernelILi32ELi32ELi2ELi2ELi3ELb1ELi0E}
SKIP=${5:-15}
mkdir -p gpurun_out
CMD="python tools/prof_hgemv.py --config $CFG --reps 2"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"$KDENSE" -c 1 -o gpurun_out/prof_dense_${CFG}_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"$KCOUP" -s $SKIP -c 1 -o gpurun_out/prof_coupling_${CFG}_$TAG $CMD > gpurun_out/ncu_full2_$TAG.log 2>&1
echo "exit $?"
tail -n 3 gpurun_out/plain_$TAG.log gpurun_out/ncu_full_$TAG.log gpurun_out/ncu_full2_$TAG.log
