#!/bin/bash
# A/B build variants: [BENCH_ARGS="--workload resnet18"] tools/ab.sh main v1 v2 ...  (libNAME.so in the package dir)
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="$PWD/paper_2509_01253_b200/lib$v.so"; fi
  tag=$(echo "$BENCH_ARGS" | tr -c 'a-z0-9' '_')
  SFHR_LIB_PATH=$lib timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/ab_$v$tag.json 2> gpurun_out/ab_$v$tag.err
  echo "$v $BENCH_ARGS rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$v$tag.json'));print(round(d['ms_per_step'],2), round(d['roofline']['kernel_ms_per_step'],2))" 2>/dev/null)"
done
