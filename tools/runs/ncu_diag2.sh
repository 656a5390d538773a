# ncu --set full of the p = 2 diagonal kernel at 160^3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diag2 --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/prof_diag2 python tools/prof_diag.py --order 2 --n 160 > gpurun_out/ncu_diag2.log 2>&1
tail -1 gpurun_out/ncu_diag2.log
