rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 26 -c 1 -o gpurun_out/r17_sweep python scripts/step_profile.py cfg2 > gpurun_out/r17_ncu.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py gpurun_out/r17_summary.md gpurun_out/r17_sweep.ncu-rep > /dev/null 2>&1
ncu -i gpurun_out/r17_sweep.ncu-rep --page details --csv > gpurun_out/r17_details.csv 2>/dev/null
ncu -i gpurun_out/r17_sweep.ncu-rep --page source --csv --print-source sass > /tmp/src.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/src.csv')))
print(len(rows))
h=rows[0]
print(h[:12])
open('gpurun_out/r17_source_head.txt','w').write('\n'.join(','.join(r) for r in rows[:2]))
# keep rows with most stall samples
idx=[i for i,c in enumerate(h) if 'Sampling' in c and 'All' in c]
print(idx)
if idx:
    j=idx[0]
    def f(r):
        try: return float(r[j])
        except: return 0
    top=sorted(rows[1:], key=lambda r:-f(r))[:80]
    with open('gpurun_out/r17_source_top.csv','w') as fo:
        w=csv.writer(fo); w.writerow(h); [w.writerow(r) for r in top]
PY
ls -la gpurun_out; rm -f gpurun_out/*.ncu-rep
cat gpurun_out/r17_summary.md
