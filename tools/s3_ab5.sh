#!/bin/bash
# session-3 A/B 5 / 7: main (working tree) vs prev (HEAD) on ResNet-20 and ResNet-18 + stage GPU tests
set -u
bash tools/ab.sh main prev main prev
BENCH_ARGS="--workload resnet18" bash tools/ab.sh main prev
timeout 900 python -m pytest tests -m gpu -x -q -k "stage or keyswitch or round or inference or misaligned" 2>&1 | tail -2
