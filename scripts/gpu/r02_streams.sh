set -x
for c in cfg2 cfg4; do for k in 1 2 3 4; do timeout 600 python bench.py --config $c --streams $k --cpu-baseline 0 > gpurun_out/st_${c}_$k.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/st_${c}_$k.json')); print('$c streams $k', round(j['value'],2), round(j['e2e']['value'],2), j['clocks']['sm_mhz'])"; done; done
