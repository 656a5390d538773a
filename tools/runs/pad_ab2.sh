# A/B: padded (default) vs dense generic-kernel sweep buffers
for r in 1 2; do
for lib in paper_2205_12721_b200/libtmop_b200.so vlibs/nopad/libtmop_b200.so; do
  echo "== $lib"
  TMOP_LIB=$lib python tools/time_phases.py --order 4 --n 80 --reps 10 | grep -E "apply|setup|gradient|diag"
  for p in 2 3 4; do TMOP_LIB=$lib python tools/time_phases.py --order $p --n 24 --nq 9 --reps 40 | grep -E "p=|apply|gradient"; done
done
done
