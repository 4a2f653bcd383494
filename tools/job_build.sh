#!/bin/bash
# Build-kernel session: build, build parity tests, Build-only A/B timing, K9 microbenchmark.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-build or bcs or categorical}" > gpurun_out/pytest_build.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_build.log
timeout 300 python tools/bench_build.py --config buildonly --modes ${MODES:-seeded,auto,global,cache} > gpurun_out/bench_build.jsonl 2>&1
timeout 120 python tools/bench_build.py --config large --modes auto,seeded >> gpurun_out/bench_build.jsonl 2>&1
timeout 120 ./tools/microbench > gpurun_out/microbench.jsonl 2>&1
