#!/bin/bash
# Merge-kernel A/B under ncu launch timing (serialised, per-launch durations summed per variant):
#   tools/ab_linear.sh "SFHR_MMA_RUN_ROWS=64" "SFHR_CONV_BLOCK=2 ..." ...
for v in "$@"; do
  tag=$(echo "$v" | tr -c "A-Za-z0-9" "_")
  env $v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:merge --csv \
    --log-file gpurun_out/mrg_$tag.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline $BENCH_ARGS > /dev/null 2>&1
  echo "$v rc=$? $(python tools/launch_summary.py gpurun_out/mrg_$tag.csv 1 2>/dev/null | head -1 | tr '\n' ' ')"
done
