for lib in paper_2205_12721_b200/libtmop_b200.so vlibs/g3/libtmop_b200.so; do
  echo "== $lib"
  for cfg in "1 200" "2 160" "3 107"; do set -- $cfg; TMOP_LIB=$lib python tools/time_phases.py --order $1 --n $2 --reps 10 | grep -E "gradient"; done
done
