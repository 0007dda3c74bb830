#!/bin/bash
# One gpurun call: build check, GPU parity tests, per-case timing, bench line,
# ncu launch list of the bench command, ncu --set full of the top kernel.
# usage (here): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests/ -m gpu -x -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python tools/perf_cases.py > $O/perf_cases.txt 2>&1; cat $O/perf_cases.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; tail -3 $O/bench.err; cat $O/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --quick --no-cpu --steps 16 --warmup 3 > $O/launches_bench.log 2>&1; tail -2 $O/launches.csv
NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 4 -c 2 \
  -o $O/prof_w3_m1_4096x14336 python tools/profile_case.py 1 4096 14336 3 128 8 > $O/ncu_w3.log 2>&1; tail -2 $O/ncu_w3.log
NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 4 -c 2 \
  -o $O/prof_w4_m1_4096x4096 python tools/profile_case.py 1 4096 4096 4 128 8 > $O/ncu_w4.log 2>&1; tail -2 $O/ncu_w4.log
NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 4 -c 1 \
  -o $O/prof_w3_m32_4096x14336 python tools/profile_case.py 32 4096 14336 3 128 8 > $O/ncu_w3m32.log 2>&1; tail -2 $O/ncu_w3m32.log
timeout 300 python tools/perf_tc.py > $O/perf_tc.txt 2>&1; cat $O/perf_tc.txt
timeout 300 python tools/perf_refine.py 4096 4096 128 > $O/perf_refine.txt 2>&1; cat $O/perf_refine.txt
