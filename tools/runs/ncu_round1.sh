# Round-1 evidence (one GPU): launch list of the default bench command's
# p=2 section, and one `ncu --set full` capture each of the x-line apply
# (bench config), the x-line setup and the diagonal at p=2 160^3.
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu --no-newton --orders 2 > gpurun_out/ncu_launches_r1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:xl_kernelILi3ELi4ELi1E -s 1 -c 1 -o gpurun_out/prof_r1_apply \
  python tools/prof_apply.py --order 2 --n 160 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:xl_kernelILi3ELi4ELi0E -s 0 -c 1 -o gpurun_out/prof_r1_setup \
  python tools/prof_apply.py --order 2 --n 160 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diag2 -s 1 -c 1 -o gpurun_out/prof_r1_diag \
  python tools/prof_diag.py --order 2 --n 160 > /dev/null 2>&1
ls -la gpurun_out/
