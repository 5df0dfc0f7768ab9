#!/bin/bash
# Round evidence on one B200 (run under gpurun): tests, smoke, ncu traffic
# captures, every bench config, the reference arm, launch lists and HARA kernel
# captures. Outputs to gpurun_out/ev/ (copied to profiles/ by hand).
set -u
O=gpurun_out/ev
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
for c in cfg2 cfg2b1; do
  timeout 900 python tools/ncu_traffic.py $c > $O/ncu_traffic_$c.log 2>&1
  cp profiles/ncu_traffic_$c.json $O/ 2>/dev/null
done
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --impl reference > $O/bench_cfg2_reference.json 2> $O/bench_cfg2_reference.err
for c in cfg2b1 cfg1 cfg4; do
  python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
python bench.py --config cfg1build --steps 3 --warmup 1 --hara-rng reference > $O/bench_cfg1build.json 2> $O/bench_cfg1build.err
python bench.py --config cfg3 --steps 3 --warmup 1 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --config cfg3 --steps 1 --warmup 1 --hara-rng reference --no-cpu-baseline > $O/bench_cfg3_refrng.json 2> $O/bench_cfg3_refrng.err
python bench.py --config cfg5 --steps 2 --warmup 1 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
# launch list of one replayed cfg2 hgemv (the 5th call: calls 1-2 eager, 3 captured, 4-5 replayed);
# only the hgemv kernels match the filter, so the setup (tree, matrix generation) is skipped
NL=$(python tools/run_hgemv.py cfg2 32 1 2>/dev/null | sed -n 's/launches per hgemv: //p')
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function \
  --kernel-name regex:"seg_gemm|gather_blocked|sym_|csr_sum" --launch-skip $((4 * NL)) --launch-count $NL \
  --csv --log-file $O/launches_cfg2.csv python tools/run_hgemv.py cfg2 32 5 > /dev/null 2>&1
for k in qr_kernel jacobi_kernel bgemm_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function --kernel-name regex:$k \
    --launch-skip 200 --launch-count 1 -f -o $O/hara_$k python tools/hara_launches.py cfg1build 1 > /dev/null 2>&1
done
# keep gpurun_out under the 64 MiB copy-back limit: summarise every ncu report, then drop it
for r in $O/*.ncu-rep gpurun_out/*.ncu-rep; do
  [ -f "$r" ] || continue
  python tools/ncu_summary.py "$r" > "${r%.ncu-rep}_summary.txt" 2>&1
  rm -f "$r"
done
du -sh gpurun_out
ls -la $O
