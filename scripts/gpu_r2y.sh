# trajectory tests (restructured), ncu launch list of the attention microbenchmark (classic vs fused backward at dh 64)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trajectory.py -q -rf -s -p no:cacheprovider > gpurun_out/r2y_traj.txt 2>&1; grep -E "200-step|const|passed|failed" gpurun_out/r2y_traj.txt
export MB_NOGRAPH=1
python scripts/microbench.py attn 16,20,1024,64 > gpurun_out/r2y_mb.txt 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2y_attn_launches.csv python scripts/microbench.py attn 16,20,1024,64 > gpurun_out/r2y_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/r2y_attn_launches.csv')))
h = None
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    if r and r[0] == 'ID': h = r; continue
    if h is None or len(r) != len(h): continue
    d = dict(zip(h, r))
    k = d['Kernel Name'][:60]
    v = float(d['Metric Value'].replace(',', ''))
    m = d['Metric Name']
    if m == 'gpu__time_duration.sum':
        agg[k][0] += 1; agg[k][1] += v
    elif 'dram' in m:
        agg[k][2] += v
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} n={n:3d} avg {t / max(n,1) / 1000:.1f} us  dram/launch {b / max(n,1) / 1e6:.1f} MB")
PY
