python bench.py --config c4 --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_surface_colored" -s 4 -c 2 \
    -o gpurun_out/prof_c4 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c4.log
