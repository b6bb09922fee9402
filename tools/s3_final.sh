#!/bin/bash
# session-3 closing checks on HEAD: full GPU tests, smoke, headline bench, primitives (NTT change)
set -u
O=gpurun_out/s3final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_resnet20.json 2> $O/bench_resnet20.err; echo "bench rc=$?"
timeout 900 python bench_primitives.py > $O/primitives.jsonl 2> $O/primitives.err; echo "primitives rc=$?"
