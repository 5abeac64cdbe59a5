python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tpe_first_pipe" -s 1 -c 1 \
    -o gpurun_out/prof_pipe python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
