#!/bin/bash
# A/B environment settings on the main build: tools/ab_env.sh "A=1" "A=0" ...
for e in "$@"; do
  tag=$(echo "$e" | tr -c 'A-Za-z0-9' '_')
  env $e timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/abenv_$tag.json 2> gpurun_out/abenv_$tag.err
  echo "$e rc=$? $(python -c "import json;d=json.load(open('gpurun_out/abenv_$tag.json'));print(round(d['ms_per_step'],2), round(d['roofline']['kernel_ms_per_step'],2))" 2>/dev/null)"
done
