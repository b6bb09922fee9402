#!/bin/bash
# Round-2 final measurement set (third session, after the MAC unroll) (one GPU call): headline bench, reference arm, other workloads,
# gamma 1 / 2 of the headline, primitives, launch list, ncu of the dominant kernel.
set -u
mkdir -p gpurun_out/r02j
O=gpurun_out/r02j
timeout 600 python bench.py > $O/bench_resnet20.json 2> $O/bench_resnet20.err; echo "resnet20 rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
for g in 1 2; do timeout 600 python bench.py --gamma $g --no-cpu-baseline > $O/bench_resnet20_g$g.json 2> $O/bench_resnet20_g$g.err; echo "g$g rc=$?"; done
for w in mlp resnet18 resnet34; do timeout 900 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"; done
timeout 900 python bench_primitives.py > $O/primitives.jsonl 2> $O/primitives.err; echo "primitives rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_resnet20.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ks_stage_kernel -s 0 -c 2 -o $O/ncu_stage python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_stage.log 2>&1; echo "ncu stage rc=$?"
ncu -i $O/ncu_stage.ncu-rep --page raw --csv > $O/ncu_stage_raw.csv 2>/dev/null; echo "raw rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
