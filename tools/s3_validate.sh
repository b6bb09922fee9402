set -u
mkdir -p gpurun_out/s3
O=gpurun_out/s3
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_resnet20.json 2> $O/bench_resnet20.err; echo "bench rc=$?"
tail -3 $O/gpu_tests.log; cat $O/bench_resnet20.json
