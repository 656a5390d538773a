# ncu --set full: the p=2 x-line apply as one whole-mesh launch (bench config) and the n_q=9 p=1 generic apply
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:xl_kernelILi3ELi4ELi1E -s 1 -c 1 -o gpurun_out/prof_r1_apply \
  python tools/prof_apply.py --order 2 --n 160 --reps 2 > gpurun_out/ncu_apply_whole.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elem_kernelILi3ELi2ELi9ELi1E --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/prof_wide_p1 python tools/prof_apply.py --order 1 --n 24 --nq 9 --reps 2 >> gpurun_out/ncu_apply_whole.log 2>&1
tail -2 gpurun_out/ncu_apply_whole.log
