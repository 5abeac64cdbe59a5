# Round profile of one config: bench line (with the paper's comparisons),
# launch list, one full ncu capture of the stage-2 color launches.
#   TAG=r1c2 CONFIG=c2 NC=3 bash tools/gpu_profile.sh
set -x
TAG=${TAG:-r1}
CONFIG=${CONFIG:-c2}
NC=${NC:-3}
python bench.py --config $CONFIG --variants > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --config $CONFIG --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --config $CONFIG --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(tpe|surface)_colored" -s $NC -c $NC \
    -o gpurun_out/prof_${TAG} python bench.py --config $CONFIG --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > gpurun_out/gpu_${TAG}.txt
