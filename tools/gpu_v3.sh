set -x
python -m pytest tests -q -m gpu -x 2>&1 | tail -4
python bench.py --no-cpu > gpurun_out/bench_v6.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/bench_v6.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_color_gbs'])"
python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_surface_colored -s 3 -c 3 -o gpurun_out/prof_v6 python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_v6.log 2>&1
