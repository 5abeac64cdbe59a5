# every config once (1 GPU): the default bench line (comparisons, CPU leg) per config
for c in ${CONFIGS:-c1 c2 c3 c5 h1 c4}; do
  python bench.py --config $c --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value']/1e9,3), 'G edges/s', round(d['ms_per_step'],3), 'ms', 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'], {k: round(v) for k,v in d['roofline']['per_color_gbs'].items()}, 'e2e', round(d['e2e']['value']/1e9,3), 'cpu', round(d['cpu_baseline']['value']/1e6,3), 'cmp', {k: round(v,3) for k,v in d.get('comparisons',{}).items() if k.endswith('_ms')})" || tail -5 gpurun_out/bench_$c.err
done
