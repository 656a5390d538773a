# ncu --set full of the n_q = 9 Hessian action (generic element kernel, p = 1 and p = 3)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elem_kernelILi3ELi2ELi9ELi1E --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/prof_wide_p1 python tools/prof_apply.py --order 1 --n 24 --nq 9 --reps 2 > gpurun_out/ncu_wide.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elem_kernelILi3ELi4ELi9ELi1E --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/prof_wide_p3 python tools/prof_apply.py --order 3 --n 24 --nq 9 --reps 2 >> gpurun_out/ncu_wide.log 2>&1
tail -2 gpurun_out/ncu_wide.log
