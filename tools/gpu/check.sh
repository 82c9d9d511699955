#!/bin/bash
# GPU check run (gpurun): pytest -m gpu, smoke(), a short N=1 bench. Logs under gpurun_out/$1/.
OUT=gpurun_out/${1:-check}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -rf --timeout 900 ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS} > $OUT/bench.log 2>&1; echo "bench rc $?"
tail -15 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; tail -c 4000 $OUT/bench.log
