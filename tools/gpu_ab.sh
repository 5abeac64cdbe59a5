# A/B harness (run through gpurun): rebuild with MC_DEFINES, run the bench
# with an environment assignment, append one summary line per run.
#   edit the loop at the bottom, then: gpurun -- 'bash tools/gpu_ab.sh'
run() {  # $1 = defines, $2 = env assignment
  MC_DEFINES="$1" python paper_1601_07613_b200/_build.py --force > /dev/null
  env $2 python bench.py --no-cpu --no-variants --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/ab.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print('[$1 | $2 | ${BENCH_ARGS}]', round(d['value']/1e9,3), 'G edges/s', round(d['ms_per_step'],3), 'ms', round(d['roofline']['frac'],3), {k: round(v) for k,v in d['roofline']['per_color_gbs'].items()})" >> gpurun_out/ab_summary.txt 2>&1 || tail -3 gpurun_out/ab.json >> gpurun_out/ab_summary.txt
}
rm -f gpurun_out/ab_summary.txt
# AB_CONFIGS / AB_DEFINES / AB_ENVS (';'-separated define sets, "" = default) select the runs
IFS=';' read -ra DEFS <<< "${AB_DEFINES:-}"
[ ${#DEFS[@]} -eq 0 ] && DEFS=("")
IFS=';' read -ra ENVS <<< "${AB_ENVS:-X=1}"     # ';'-separated env assignments
for cfg in ${AB_CONFIGS:-c2}; do export BENCH_ARGS="--config $cfg --steps ${AB_STEPS:-10}"
  for d in "${DEFS[@]}"; do for e in "${ENVS[@]}"; do run "$d" "$e"; done; done; done
cat gpurun_out/ab_summary.txt
