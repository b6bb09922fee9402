#!/bin/bash
# session-3 A/B: stage kernel variants (ResNet-20 and ResNet-18) + stage-kernel GPU tests
set -u
bash tools/ab.sh main nobulk bulkonly main nobulk
BENCH_ARGS="--workload resnet18" bash tools/ab.sh main nobulk
timeout 900 python -m pytest tests -m gpu -x -q -k "stage or keyswitch or round or inference" 2>&1 | tail -3
