#!/bin/bash
# ncu captures of the build kernel (seeded and table pi) on Build-only.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python tools/bench_build.py --config buildonly --modes seeded,auto --iters 2 > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:build_kernel -s 3 -c 1 -o gpurun_out/${TAG:-r02_build}_seeded -f \
    python tools/bench_build.py --config buildonly --modes seeded --iters 2 > gpurun_out/ncu_seeded.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:build_kernel -s 3 -c 1 -o gpurun_out/${TAG:-r02_build}_table -f \
    python tools/bench_build.py --config buildonly --modes auto --iters 2 > gpurun_out/ncu_table.log 2>&1
