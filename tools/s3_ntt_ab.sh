#!/bin/bash
# session-3 NTT A/B: batched global / DSMEM loads (NTT_BATCH_IO bits) per variant library
mkdir -p gpurun_out/s3
for v in ${NTT_VARIANTS:-main nio0 nio2 main}; do
  if [ "$v" = main ]; then lib=""; else lib="$PWD/paper_2509_01253_b200/lib$v.so"; fi
  SFHR_LIB_PATH=$lib timeout 300 python bench_primitives.py --sections ntt > gpurun_out/s3/ntt_$v.jsonl 2>gpurun_out/s3/ntt_$v.err; echo "$v rc=$?"
done
timeout 300 python -m pytest tests/test_ntt64.py -x -q 2>&1 | tail -2
