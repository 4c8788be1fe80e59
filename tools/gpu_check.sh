#!/bin/bash
# Quick GPU check (run on the GPU box from the repo root; outputs in gpurun_out/):
# GPU tests (minus the BASELINE-scale fixtures unless SCALE=1), smoke, default bench.
set -u
O=gpurun_out/chk
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
if [ "${SCALE:-0}" = "1" ]; then SEL=""; else SEL="--ignore=tests/test_gpu_scale.py"; fi
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q $SEL ${PYTEST_ARGS:-} > $O/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
  tail -c 600 $O/bench.err
fi
