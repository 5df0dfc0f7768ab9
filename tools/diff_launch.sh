export PATH=/usr/local/cuda/bin:$PATH
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/diff_launches.csv python tools/diff1d_probe.py --b 16 --reps 1 --check 0 --tune 16:64:0 > gpurun_out/diff_ncu1.log 2>&1
