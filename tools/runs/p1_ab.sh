timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for lib in paper_2205_12721_b200/libtmop_b200.so vlibs/p1mb4/libtmop_b200.so; do echo "== $lib"; for i in 1 2; do TMOP_LIB=$lib python tools/time_apply.py --order 1 --n 200 --steps 10 | tail -1; done; done
