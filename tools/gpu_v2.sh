set -x
python -m pytest tests -q -m gpu -x 2>&1 | tail -4
python bench.py --no-cpu > gpurun_out/bench_v2_minb3.json 2>&1; cat gpurun_out/bench_v2_minb3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_color_gbs'])"
MC_DEFINES="MC_MINB_2D=2" python paper_1601_07613_b200/_build.py --force
python bench.py --no-cpu --variants > gpurun_out/bench_v2_minb2.json 2>&1; cat gpurun_out/bench_v2_minb2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_color_gbs'], d.get('comparisons'))"
