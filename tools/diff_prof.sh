# ncu evidence for the device diffusion Hessian (tools/diff1d_probe.py at cfg3 size, b=16)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:cn_step_kernel --launch-skip 100 -c 1 -o gpurun_out/diff_step1 python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cn_step_kernel --launch-skip 180 -c 1 -o gpurun_out/diff_step2 python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_ncu3.log 2>&1
