# ncu evidence for the device diffusion Hessian (tools/diff1d_probe.py at cfg3 size, b=16, multi-kernel path)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:cn_step_kernel --launch-skip 120 -c 1 -o gpurun_out/diff_step python tools/diff1d_probe.py --b 16 --reps 1 --check 0 --tune 16:64:0 > gpurun_out/diff_ncu2.log 2>&1
