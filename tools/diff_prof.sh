# ncu evidence for the device diffusion Hessian (tools/diff1d_probe.py at cfg3 size, b=16)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/diff_launches.csv python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cn_step_kernel --launch-skip 300 -c 1 -o gpurun_out/diff_step python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_ncu2.log 2>&1
ncu --set full --clock-control none -k regex:carry_fwd_scan --launch-skip 300 -c 1 -o gpurun_out/diff_carry python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_ncu3.log 2>&1
