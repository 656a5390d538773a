# n_q = 9 operator phases after the L2-prefetch / per-kind occupancy change
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for p in 1 2 3 4; do python tools/time_phases.py --order $p --n 24 --nq 9 --reps 20; done
