set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
for p in 1 2; do
  n=$([ $p = 1 ] && echo 200 || echo 160)
  timeout 120 python tools/time_apply.py --order $p --n $n --steps 10
  TMOP_APPLY_KERNEL=generic timeout 120 python tools/time_apply.py --order $p --n $n --steps 10
done
