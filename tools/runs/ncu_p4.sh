# ncu --set full of the p = 4 generic-element apply (n_q = 6) at 80^3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elem_kernelILi3ELi5ELi6ELi1E --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/prof_p4b python tools/prof_apply.py --order 4 --n 80 --reps 2 > gpurun_out/ncu_p4b.log 2>&1
tail -1 gpurun_out/ncu_p4b.log
