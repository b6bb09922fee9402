#!/bin/bash
# A/B NTT build variants: tools/ab_ntt.sh main v1 ...
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="$PWD/paper_2509_01253_b200/lib$v.so"; fi
  SFHR_LIB_PATH=$lib timeout 600 python bench_primitives.py --sections ntt --quick > gpurun_out/abntt_$v.jsonl 2> gpurun_out/abntt_$v.err
  echo "$v rc=$? $(python -c "
import json
for l in open('gpurun_out/abntt_$v.jsonl'):
    d=json.loads(l)
    if d.get('section')=='ntt' and d['batch']==64 and d['L'] in (16,) : print(d['op'][:3], d['N'], d['GB/s'], end=' | ')
")"
done
