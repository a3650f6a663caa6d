#!/bin/bash
# Quick GPU iteration: GPU tests, then c4 (and optionally c1) bench without the CPU baseline.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout ${TTMO:-900} python -m pytest tests -m gpu -x -q ${PYARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-4 1}; do
  BENCH_NO_CPU=1 timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print('c$c', d['value'], d['unit'], d['ms_per_step'], 'frac', d['roofline']['frac'], 'cg/p', d['cg_iters_per_problem'], 'op', d['operator'])" || tail -20 gpurun_out/bench_c$c.err
done
