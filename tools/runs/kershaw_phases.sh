# operator phase timings at the paper's Kershaw sizes (24^3, n_q = 9)
for p in 1 2 3 4; do python tools/time_phases.py --order $p --n 24 --nq 9 --reps 20; done
