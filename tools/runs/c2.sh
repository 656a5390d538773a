# C2 apply timings and the launch list
python tools/time_c2.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python tools/time_c2.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:xl_kernelILi2ELi3ELi8E --kernel-name-base mangled -s 10 -c 1 -o gpurun_out/prof_c2 python tools/time_c2.py > /dev/null 2>&1
ls gpurun_out
