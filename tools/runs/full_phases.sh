# full GPU suite + phase timings at p=2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python tools/time_phases.py --order 2 --n 160
python tools/time_phases.py --order 3 --n 100
