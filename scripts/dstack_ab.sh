# Same-box A/B of persistent-decode variants: the in-tree build vs build/ab/<name> for each name given,
# alternating twice (timeline medians, scripts/dstack_trace.py)
for rep in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then R=""; else R="build/ab/$v"; fi
    echo "== $v"; DS_PKG_ROOT=$R timeout 300 python scripts/dstack_trace.py 2>&1 | grep -E "us/token|^A |^B |bar A|bar B|bar C|^C |^layer |A epi units"
  done
done
