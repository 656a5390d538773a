timeout 900 python -m pytest tests -x -q -m gpu -k "padded or oracle or kershaw" 2>&1 | tail -2
for r in 1 2; do
for lib in paper_2205_12721_b200/libtmop_b200.so vlibs/noring/libtmop_b200.so; do
  echo "== $lib"
  for p in 1 2 3 4; do TMOP_LIB=$lib python tools/time_phases.py --order $p --n 24 --nq 9 --reps 40 | grep -E "apply"; done
done; done
