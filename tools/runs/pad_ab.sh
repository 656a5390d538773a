# padded generic-kernel sweep buffers: GPU suite + p=4 (n_q=6) and n_q=9 phase timings
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/time_phases.py --order 4 --n 80 --reps 10
for p in 1 2 3 4; do python tools/time_phases.py --order $p --n 24 --nq 9 --reps 20 | grep -E "p=|apply|setup|gradient"; done
