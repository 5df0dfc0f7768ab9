export PATH=/usr/local/cuda/bin:$PATH
python tools/hara_launches.py cfg3k > gpurun_out/hara_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/hara_launches.csv python tools/hara_launches.py cfg3k > gpurun_out/hara_ncu.log 2>&1
