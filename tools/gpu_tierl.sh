#!/bin/bash
# Tier L quick check: grid-tier GPU tests, then c5 / c3 / c2 timings and the c5 operator.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_recover.py tests/test_gpu_operator.py tests/test_gpu_cg_counts.py tests/test_gpu_topk.py -q -x ${PYARGS} 2>&1 | tail -4
for c in ${CONFIGS:-5 3 2}; do
  BENCH_NO_CPU=1 timeout 600 python bench.py --config $c --steps 3 --warmup 2 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); o=d['operator']; print('c$c', d['ms_per_step'], 'ms', 'cg', d['cg_iters_per_problem'], 'outer', d['outer_iters_mean'], 'op fwd/adj ms', round(o['ms_fwd'],4), round(o['ms_adj'],4), 'frac', round(o['frac_hbm_fwd'],3), round(o['frac_hbm_adj'],3))" || tail -5 gpurun_out/bench_c$c.err
done
