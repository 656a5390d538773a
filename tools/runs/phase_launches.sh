# per-launch device times of every operator entry point at p=2 n=160
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/phase_launches.csv python tools/time_phases.py --order 2 --n 160 --reps 1 > gpurun_out/phase_launches.log 2>&1
tail -3 gpurun_out/phase_launches.log
