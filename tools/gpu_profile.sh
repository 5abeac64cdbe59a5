# Round profile of one config: bench line (default: with the paper's
# comparisons and the CPU leg), launch list, one full ncu capture of the
# stage-2 color launches of the first warm-up step.
#   TAG=r2c4a CONFIG=c4 NC=4 bash tools/gpu_profile.sh
set -x
TAG=${TAG:-r2}
CONFIG=${CONFIG:-c4}
NC=${NC:-4}
QUICK="--config $CONFIG --steps 1 --warmup 3 --no-cpu --no-variants --e2e-steps 1"
[ -n "$NO_BENCH" ] || python bench.py --config $CONFIG > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py $QUICK > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py $QUICK > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(tpe|surface)_colored" -s $NC -c $NC \
    -o gpurun_out/prof_${TAG} python bench.py $QUICK > gpurun_out/ncu_full_${TAG}.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > gpurun_out/gpu_${TAG}.txt
