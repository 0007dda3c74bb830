O=gpurun_out/d6; mkdir -p $O
NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 2 -c 1 -o $O/w1 python tools/profile_case.py 1 4096 4096 4 128 3 1 > $O/w1.log 2>&1; tail -1 $O/w1.log
export FLUTE_LIB=paper_2407_10960_b200/libflute_b200_diag.so
FLUTE_DIAG=15 NCU_PROFILING=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm -s 2 -c 1 -o $O/w1_d15 python tools/profile_case.py 1 4096 4096 4 128 3 1 > $O/w1d.log 2>&1; tail -1 $O/w1d.log
