# ncu --set full of the p = 1 x-line apply (n_q = 3) at 200^3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xl_kernelILi2ELi3ELi1E --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/prof_p1b python tools/prof_apply.py --order 1 --n 200 --reps 2 > gpurun_out/ncu_p1b.log 2>&1
tail -1 gpurun_out/ncu_p1b.log
