#!/bin/bash
# session-3 A/B 5: prologue copies issued before the barrier-init CTA barrier (main) vs previous HEAD (prev)
set -u
bash tools/ab.sh main prev main prev
BENCH_ARGS="--workload resnet18" bash tools/ab.sh main prev
timeout 900 python -m pytest tests -m gpu -x -q -k "stage or keyswitch or round or inference or misaligned" 2>&1 | tail -2
