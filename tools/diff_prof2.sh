# ncu of the persistent diffusion march (tools/diff1d_probe.py --b 1, N=2^18, steps 64)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
python tools/diff1d_probe.py --b 1 2 3 --check 0 > gpurun_out/diffp_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cn_march_kernel --launch-skip 1 -c 1 -o gpurun_out/diff_march python tools/diff1d_probe.py --b 1 --reps 1 --check 0 > gpurun_out/diffp_ncu.log 2>&1
