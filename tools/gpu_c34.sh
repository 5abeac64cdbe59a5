python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for c in c2 c3 c4; do
  python bench.py --config $c --steps 10 --no-cpu --e2e-steps 1 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value']/1e9,3), 'G edges/s', round(d['ms_per_step'],3), 'ms', 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'], {k: round(v) for k,v in d['roofline']['per_color_gbs'].items()})" || tail -5 gpurun_out/bench_$c.err
done
