set -x
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_probe tools/dmma_probe.cu && /tmp/dmma_probe
python -m pytest tests -q -m gpu -x 2>&1 | tail -4
python bench.py --no-cpu > gpurun_out/bench_v13.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/bench_v13.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_color_gbs'])"
python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_(tpe|surface)_colored" -s 3 -c 3 -o gpurun_out/prof_v13 python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_v13.log 2>&1
