#!/bin/bash
# Full verification session: GPU suite, whole-output parity, bench, launch list, top-k ncu capture.
mkdir -p gpurun_out
T=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_gpu.txt 2>&1
nproc > gpurun_out/${T}_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/${T}_host.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
if [ -n "$FULLPAR" ]; then
  BSK_FULL_PARITY=1 timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -s > gpurun_out/${T}_parity_large_full.log 2>&1
  echo "full parity exit $?" >> gpurun_out/${T}_parity_large_full.log
fi
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench.log
if [ -n "$NCU" ]; then
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/${T}_bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_large.csv \
      python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/${T}_ncu_launches.log 2>&1
  python tools/bench_topk.py --config large --iters 1 --warmup 1 > gpurun_out/${T}_topk_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:tc_pairs_kernel -s 1 -c 1 -o gpurun_out/${T}_topk_final -f \
      python tools/bench_topk.py --config large --iters 1 --warmup 1 > gpurun_out/${T}_ncu_topk.log 2>&1
fi
