# Round profile: plain bench, launch list, one full capture of the colored kernel.
set -x
TAG=${TAG:-r1}
python bench.py --variants > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(tpe|surface)_colored" -s 3 -c 3 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > gpurun_out/gpu_${TAG}.txt
