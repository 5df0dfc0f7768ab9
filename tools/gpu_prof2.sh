#!/bin/bash
# ncu evidence round 1 v2: cfg2 launch list + dense/coupling kernels, cfg2b1 dense block pass
mkdir -p gpurun_out
C2="python tools/prof_hgemv.py --config cfg2 --reps 2"
C1="python tools/prof_hgemv.py --config cfg2b1 --reps 2"
$C2 > gpurun_out/plain_v2.log 2>&1 && $C1 >> gpurun_out/plain_v2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_r01v2.csv $C2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'seg_gemm_kernelILi64ELi32ELi2ELi2ELi2ELi32ELb1ELi2E' -c 1 -o gpurun_out/prof_dense_cfg2_r01v2 $C2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'sym_pass64_kernel' -c 1 -o gpurun_out/prof_sympass64_cfg2b1_r01v2 $C1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'sym_pass32_kernel' -c 1 -o gpurun_out/prof_sympass32_cfg2b1_r01v2 $C1 > /dev/null 2>&1
echo "exit $?"
