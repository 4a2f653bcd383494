#!/bin/bash
# Top-k A/B: full GPU test suite on the default library, then Large top-k timing per variant.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 200 python tools/bench_topk.py --config large --iters 2 > gpurun_out/quick.log 2>&1 || { echo "quick check failed" >> gpurun_out/quick.log; exit 1; }
if [ -z "$NOTEST" ]; then
if [ -n "$PYTEST_K" ]; then timeout 1200 python -m pytest tests -m gpu -q -x --timeout=300 -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 1200 python -m pytest tests -m gpu -q -x --timeout=300 > gpurun_out/pytest_gpu.log 2>&1; fi
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
for v in default ${VARIANTS}; do
  if [ "$v" = default ]; then unset BINSKETCH_LIB_VARIANT; else export BINSKETCH_LIB_VARIANT=$PWD/variants/libbinsketch_$v.so; fi
  echo "== $v" >> gpurun_out/topk_ab.jsonl
  timeout 300 python tools/bench_topk.py --config ${CONFIG:-large} ${TOPK_ARGS} >> gpurun_out/topk_ab.jsonl 2>&1
done
