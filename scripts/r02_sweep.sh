# A/B sweep of a planner switch: CNN time per value (mode 5)
VAR=$1; shift
for V in "$@"; do
  echo "== $VAR=$V"
  env $VAR=$V timeout 300 python scripts/cnn_time.py 5 2>&1 | tail -1
done
