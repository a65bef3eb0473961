#!/bin/bash
# One gpurun call: GPU tests, default bench line, mgpu path at N=1, ncu
# launch list + full capture of the bench's dominant kernel.
# usage: bash scripts/gpu_check.sh TAG
TAG=${1:-x}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu_$TAG.log 2>&1; tail -2 $O/pytest_gpu_$TAG.log
timeout 300 python bench.py --steps 200 --warmup 5 --cpu-seconds 5 > $O/bench_$TAG.log 2>&1
timeout 300 python bench.py --mgpu --steps 50 --warmup 3 --e2e-steps 2 > $O/bench_mgpu_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_$TAG.csv python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:symv -s 4 -c 2 -o $O/prof_bench_$TAG python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
grep -h '^{' $O/bench_$TAG.log $O/bench_mgpu_$TAG.log | cut -c1-400
