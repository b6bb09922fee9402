#!/bin/bash
# A/B the stage-kernel build variants: tools/ab.sh name1 name2 ...  (libNAME.so in the package dir)
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="$PWD/paper_2509_01253_b200/lib$v.so"; fi
  SFHR_LIB_PATH=$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  echo "$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print(round(d['ms_per_step'],2), round(d['roofline']['kernel_ms_per_step'],2))" 2>/dev/null)"
done
