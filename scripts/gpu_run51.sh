export STN_TMA_MIN_BITS=6
STN_TMA_DBG=32 timeout 300 python scripts/ncu_target.py cfg2 1 > /tmp/w.txt 2>&1
python3 - <<'PY'
import re
lines=[l for l in open('/tmp/w.txt') if l.startswith('cta0')]
# group consecutive blocks by launch: a new launch starts when warp numbers repeat
groups=[]; cur=[]; seen=set()
for l in lines:
    w=int(l.split()[2].rstrip(':'))
    if w in seen: groups.append(cur); cur=[]; seen=set()
    seen.add(w); cur.append(l)
groups.append(cur)
groups.sort(key=lambda g: -max(int(re.search(r'total (\d+)',l).group(1)) for l in g))
for g in groups[:2]:
    print('----')
    for l in sorted(g, key=lambda l:int(l.split()[2].rstrip(':'))): print(l.rstrip())
PY
