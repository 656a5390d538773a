# non-template metric rewrite: GPU suite + C2 timings
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/time_c2.py
python tools/time_c2.py
