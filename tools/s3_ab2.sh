#!/bin/bash
# session-3 A/B 2: rows per CTA with next-row mask prefetch
set -u
bash tools/ab.sh main rows2 rows2np main rows2
BENCH_ARGS="--workload resnet18" bash tools/ab.sh main rows2
SFHR_LIB_PATH=$PWD/paper_2509_01253_b200/librows2.so timeout 900 python -m pytest tests -m gpu -x -q -k "stage or keyswitch or round or inference" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "stage or keyswitch or round or inference" 2>&1 | tail -2
