#!/bin/bash
# One measurement round on the GPU box (run from the repo root under gpurun):
#   bench line (no profiler), the bench's launch list under ncu, and ncu --set
#   full captures of the two dominant kernels (k_cg at C4, ks_solve on the
#   bench batch), summarised with tools/launch_summary.py / tools/ncu_summary.py.
# usage: tools/measure_round.sh <tag>
tag=${1:-rXX}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py > $out/${tag}_bench_line.json 2> $out/${tag}_bench.err
echo "bench rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 > $out/${tag}_ncu_launches.log 2>&1
echo "launches rc $?"
python tools/launch_summary.py $out/${tag}_launches.csv > $out/${tag}_launches_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg -s 1 -c 1 \
  -o $out/${tag}_k_cg_C4 -f python tools/prof_single.py C4 > $out/${tag}_ncu_kcg.log 2>&1
echo "ncu k_cg rc $?"
python tools/ncu_summary.py $out/${tag}_k_cg_C4.ncu-rep > $out/${tag}_ncu_k_cg_C4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ks_solve -s 1 -c 1 \
  -o $out/${tag}_ks_solve -f python tools/prof_batch.py 2000 256 2 > $out/${tag}_ncu_ks.log 2>&1
echo "ncu ks_solve rc $?"
python tools/ncu_summary.py $out/${tag}_ks_solve.ncu-rep > $out/${tag}_ncu_ks_solve.txt 2>&1
ls -la $out | tail -20
