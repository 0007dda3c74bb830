set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --quick --no-cpu --steps 16 --warmup 3 > /dev/null 2>&1; tail -5 gpurun_out/launches1.csv
NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 4 -c 2 -o gpurun_out/prof_w3_m1 python tools/profile_case.py 1 4096 14336 3 128 8 > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log
NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 4 -c 2 -o gpurun_out/prof_w4_m1 python tools/profile_case.py 1 4096 4096 4 128 8 > gpurun_out/ncu2.log 2>&1; tail -3 gpurun_out/ncu2.log
for c in "1 4096 4096 4 128" "16 4096 4096 4 128" "1 4096 14336 3 128" "32 4096 14336 3 128" "1 14336 4096 3 128"; do python tools/profile_case.py $c; done
