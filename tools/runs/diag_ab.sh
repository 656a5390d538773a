# diagonal kernel check: diag parity tests + phase timings at p=1..4
timeout 300 python -m pytest tests -x -q -m gpu -k "diag" 2>&1 | tail -2
python tools/time_phases.py --order 2 --n 160
python tools/time_phases.py --order 1 --n 200 | grep -i diag
python tools/time_phases.py --order 3 --n 100 | grep -i diag
python tools/time_phases.py --order 4 --n 80 | grep -i diag
