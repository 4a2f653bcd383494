#!/bin/bash
# Final verification session: GPU suite (with the full-size tests), smoke, whole-output Large parity,
# every bench line, launch lists, the Large top-k ncu capture, and the secondary workloads.
T=gpurun_out/${TAG:-r02_final}
mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $T/gpu.txt 2>&1
nproc > $T/host.txt; grep -m1 "model name" /proc/cpuinfo >> $T/host.txt
python -c "import __graft_entry__ as g; g.build()" > $T/build.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 > $T/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1; echo "smoke exit $?" >> $T/smoke.log
BSK_FULL_PARITY=1 timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -s > $T/parity_large_full.log 2>&1; echo "full parity exit $?" >> $T/parity_large_full.log
timeout 900 python bench.py > $T/bench_large.log 2>&1; echo "bench exit $?" >> $T/bench_large.log
timeout 600 python bench.py --workload ranking > $T/bench_ranking.log 2>&1; echo "bench exit $?" >> $T/bench_ranking.log
timeout 300 python bench.py --workload tiny > $T/bench_tiny.log 2>&1; echo "bench exit $?" >> $T/bench_tiny.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $T/bench_reference.log 2>&1; echo "bench exit $?" >> $T/bench_reference.log
timeout 600 python tools/bench_build.py --config buildonly --modes seeded,auto > $T/build_buildonly.jsonl 2>&1
timeout 600 python tools/bench_estimate.py > $T/estimate_medium.jsonl 2>&1
timeout 600 python tools/bench_join.py > $T/join_exp2.jsonl 2>&1
timeout 600 python tools/bench_mse.py --Ns 1000 --measures js,ip > $T/mse_exp1.jsonl 2>&1
timeout 300 python tools/bench_categorical.py > $T/categorical.jsonl 2>&1
timeout 300 python tools/bench_build.py --config buildonly --modes seeded,auto --bcs > $T/build_bcs.jsonl 2>&1
timeout 300 python tools/bench_pairs.py > $T/pairs_engines.jsonl 2>&1
python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > $T/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_large.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > $T/ncu_launches.log 2>&1
python tools/launch_summary.py $T/launches_large.csv > $T/launches_large_summary.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $T/launches_ranking.csv \
    python bench.py --workload ranking --steps 3 --warmup 3 --no-cpu-baseline > $T/ncu_launches_ranking.log 2>&1
python tools/launch_summary.py $T/launches_ranking.csv > $T/launches_ranking_summary.txt 2>&1
python tools/bench_topk.py --config large --iters 1 --warmup 1 > $T/topk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_pairs_kernel -s 1 -c 1 -o $T/topk_large -f \
    python tools/bench_topk.py --config large --iters 1 --warmup 1 > $T/ncu_topk.log 2>&1
echo done > $T/done.txt
