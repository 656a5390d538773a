# quick GPU check: parity tests, apply timings p=1,2, ncu of the x-line kernel at p=2 (tag = $1)
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do python tools/time_apply.py --order 2 --n 160 --steps 10; done
python tools/time_apply.py --order 1 --n 200 --steps 10
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xl_kernelILi3ELi4ELi1E --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/prof_$1 python tools/prof_apply.py --order 2 --n 80 --reps 2 > gpurun_out/ncu_$1.log 2>&1
tail -1 gpurun_out/ncu_$1.log
