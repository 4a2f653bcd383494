#!/bin/bash
# ncu capture of the fused top-k kernel at the Large config (one launch).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python tools/bench_topk.py --config large --iters 1 --warmup 1 > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:tc_pairs_kernel -s 1 -c 1 -o gpurun_out/${TAG:-r02_topk} -f \
    python tools/bench_topk.py --config large --iters 1 --warmup 1 > gpurun_out/ncu_topk.log 2>&1
