for v in base "$@"; do
  if [ $v = base ]; then R=""; else R="build/ab/$v"; fi
  echo "== $v"; DS_PKG_ROOT=$R timeout 300 python scripts/prefill_time.py --reps 5 2>&1 | grep -E "scan|dt_proj|sum"
done
