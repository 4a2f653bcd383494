#!/bin/bash
# Secondary workloads (every TC mode + the build variants) after a kernel change: timings + sampled parity.
mkdir -p gpurun_out
T=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/bench_estimate.py > gpurun_out/${T}_estimate_medium.jsonl 2>&1
timeout 600 python tools/bench_join.py > gpurun_out/${T}_join_exp2.jsonl 2>&1
timeout 600 python tools/bench_mse.py --Ns 1000 --measures js,ip > gpurun_out/${T}_mse_exp1.jsonl 2>&1
timeout 300 python tools/bench_categorical.py > gpurun_out/${T}_categorical.jsonl 2>&1
timeout 300 python tools/bench_build.py --config buildonly --modes seeded,auto --bcs > gpurun_out/${T}_build_bcs.jsonl 2>&1
timeout 300 python tools/bench_pairs.py > gpurun_out/${T}_pairs_engines.jsonl 2>&1
