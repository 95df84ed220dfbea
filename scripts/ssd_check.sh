# Mamba-2 scan iteration check: parity tests, bench line (TTFT / TPOT), per-kernel times of one layer pair
timeout 600 python -m pytest tests/test_gpu_mamba2.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --config mamba2-2.7b --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/m2_check.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/m2_check.json')); print(round(d['value']), round(d['ttft_ms'],1), round(d['tpot_ms'],3))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --config mamba2-2.7b --steps 1 --warmup 1 --no-cpu --no-e2e --layers 2 2>/dev/null > gpurun_out/m2_launches.csv
python - <<'P'
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/m2_launches.csv')) if len(r) > 10 and r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    k = (r[4][:70], r[7])
    agg.setdefault(k, []).append(float(r[-1]) / 1000)
for (n, g), v in agg.items():
    if any(x in n for x in ('elementwise', 'gather', 'index_', 'Functor', 'reduce_kernel')):
        continue
    print(f"{len(v):3d} x {sum(v)/len(v):9.1f} us  grid {g:14s} {n}")
P
