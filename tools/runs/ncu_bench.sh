# ncu evidence for the bench config (p=2, 160^3): one --set full capture of
# the Hessian-action element kernel, and the launch list of a short bench run.
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:xl_kernelILi3ELi4ELi1E -s 1 -c 1 -o gpurun_out/prof_bench_apply \
  python tools/prof_apply.py --order 2 --n 160 --reps 2 > gpurun_out/ncu_bench_apply.log 2>&1
tail -2 gpurun_out/ncu_bench_apply.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --orders 2 > gpurun_out/ncu_launches.log 2>&1
tail -2 gpurun_out/ncu_launches.log
