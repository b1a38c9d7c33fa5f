#!/bin/bash
# Round-end GPU pass (run under gpurun): GPU tests, smoke, the default bench,
# the bench's kernel launch list (ncu, durations only) and one full ncu
# capture of the dominant kernel.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "EXIT=$? SECONDS=$(( $(date +%s) - T0 ))" >> gpurun_out/bench_final.log
if grep -q '^EXIT=0' gpurun_out/bench_final.log; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
      python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:splits_sweep -c 1 \
      -o gpurun_out/sweep_full python tools/prof_splits.py > gpurun_out/ncu_sweep.log 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:side_tables -c 1 \
      -o gpurun_out/tables_full python tools/prof_splits.py > gpurun_out/ncu_tables.log 2>&1
fi
