#!/bin/bash
# One gpurun call: the round's bench evidence (default line + reference arm),
# the ncu launch list of the bench command and one `ncu --set full` capture
# of its dominant kernel.  Output under gpurun_out/, tagged.
# usage: bash scripts/round_evidence.sh TAG
TAG=${1:-x}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi_$TAG.txt 2>&1
timeout 900 python bench.py > $O/bench_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 4 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:symv_kernel -s 2 -c 2 -o $O/prof_bench_$TAG \
  python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
grep -h '^{' $O/bench_$TAG.log $O/bench_ref_$TAG.log | cut -c1-300
