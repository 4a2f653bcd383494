#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 120 python tools/bench_build.py --config large --modes auto,seeded --iters 2 > gpurun_out/quick.log 2>&1 || { echo "quick check failed" >> gpurun_out/quick.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x --timeout=120 -k "${PYTEST_K:-build or bcs or categorical}" > gpurun_out/pytest_build.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_build.log
for v in default ${VARIANTS}; do
  if [ "$v" = default ]; then unset BINSKETCH_LIB_VARIANT; else export BINSKETCH_LIB_VARIANT=$PWD/variants/libbinsketch_$v.so; fi
  echo "== $v" >> gpurun_out/bench_build_ab.jsonl
  timeout 120 python tools/bench_build.py --config buildonly --modes ${MODES:-seeded,auto} >> gpurun_out/bench_build_ab.jsonl 2>&1
done
