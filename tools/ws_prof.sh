CMD="python tools/prof_hgemv.py --config cfg2 --reps 2 --tune 0,0,2"
$CMD > gpurun_out/plain_ws.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'ws_gemm_kernelILi64ELi32ELi2ELi2ELi2ELi2E' -c 1 -o gpurun_out/prof_ws_dense $CMD > gpurun_out/ncu_ws.log 2>&1; echo done $?
