O=gpurun_out/n2; mkdir -p $O
NCU_PROFILING=1 timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:qgemm -s 6 -c 1 -o $O/w3m1 python tools/profile_case.py 1 4096 14336 3 128 8 > $O/l1.log 2>&1; tail -1 $O/l1.log
NCU_PROFILING=1 timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:qgemm -s 6 -c 1 -o $O/w3m32 python tools/profile_case.py 32 4096 14336 3 128 8 > $O/l2.log 2>&1; tail -1 $O/l2.log
