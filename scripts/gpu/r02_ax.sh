set -x
for c in cfg5 cfg4 cfg2; do timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_ax.json 2> gpurun_out/bench_${c}_ax.err; python -c "
import json; j=json.load(open('gpurun_out/bench_${c}_ax.json')); r=j['roofline']; print('$c', j['value'], j['ms_per_step'], j['e2e']['value'], r['kernel'], round(r['frac'],3), r['share_of_step'], j['arena_bytes_per_slice']/2**30, j['clocks'], {k:round(v['ms_per_step'],1) for k,v in r['per_kernel_class'].items()})"; done
