#!/bin/bash
# Bench lines for the round: default (c4 + cpu_baseline + parity), reference arm, the other configs,
# fp64 lines, the per-GPU share of the 8-GPU split (512 problems).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps ${RSTEPS:-5} --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for b in 2048 1024 512; do
  BENCH_NO_CPU=1 timeout 300 python bench.py --batch $b --steps 10 --warmup 3 --no-op-bench > gpurun_out/bench_c4_b$b.json 2> gpurun_out/bench_c4_b$b.err
done
BENCH_NO_CPU=1 timeout 600 python bench.py --precision fp64 --steps 5 --warmup 3 > gpurun_out/bench_c4_fp64.json 2> gpurun_out/bench_c4_fp64.err
for c in 1 2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
for c in 3 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
BENCH_NO_CPU=1 timeout 600 python bench.py --config 5 --precision fp64 --tol 1e-10 --steps 3 --warmup 3 > gpurun_out/bench_c5_fp64.json 2> gpurun_out/bench_c5_fp64.err
BENCH_NO_CPU=1 timeout 600 python bench.py --config 2 --precision fp64 --steps 3 --warmup 3 > gpurun_out/bench_c2_fp64.json 2> gpurun_out/bench_c2_fp64.err
for f in gpurun_out/bench_*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ['impl','value','unit','ms_per_step','dtype','scaling']}, 'roof', {k:d.get('roofline',{}).get(k) for k in ['bound','achieved','frac']} if d.get('roofline') else None)
print('  cpu', d.get('cpu_baseline')); print('  parity', d.get('parity')); print('  e2e', d.get('e2e',{}).get('value'), 'op', {k:round(v,4) for k,v in (d.get('operator') or {}).items()})
" 2>&1 | head -5; done
