timeout 900 python -m pytest tests -x -q -m gpu -k "diag or oracle or golden or padded or c3_size" 2>&1 | tail -2
for r in 1 2; do
for lib in paper_2205_12721_b200/libtmop_b200.so vlibs/nosplit/libtmop_b200.so; do
  echo "== $lib"
  TMOP_LIB=$lib python tools/time_phases.py --order 2 --n 160 --reps 10 | grep diag
  TMOP_LIB=$lib python tools/time_phases.py --order 1 --n 200 --reps 10 | grep diag
  TMOP_LIB=$lib python tools/time_phases.py --order 3 --n 107 --reps 10 | grep diag
  TMOP_LIB=$lib python tools/time_phases.py --order 4 --n 80 --reps 10 | grep diag
  TMOP_LIB=$lib python tools/time_phases.py --order 2 --n 24 --nq 9 --reps 20 | grep diag
done; done
