mkdir -p gpurun_out
for c in cfg1 cfg2b1 cfg2; do
timeout 600 python tools/order_probe.py --config $c --combos 1:0:0,1:0:1,1:0:2,1:0:0,1:0:2 > gpurun_out/fuse_$c.txt 2>&1
done
