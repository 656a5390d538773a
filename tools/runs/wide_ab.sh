# n_q = 9 Hessian action: TMA-staged Q-data vs direct loads (2 / 3 CTAs per SM)
timeout 300 python -m pytest tests -x -q -m gpu -k "apply or hessian" 2>&1 | tail -2
for lib in paper_2205_12721_b200/libtmop_b200.so vlibs/tma/libtmop_b200.so vlibs/ldg3/libtmop_b200.so; do
  echo "== $lib"
  for p in 1 2 3 4; do TMOP_LIB=$lib python tools/time_phases.py --order $p --n 24 --nq 9 --reps 20 | grep -E "p=|apply|setup"; done
done
