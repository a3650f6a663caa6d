#!/bin/bash
# Bench every BASELINE config once (no CPU baseline), for the per-config table.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in ${CONFIGS:-1 2 3 5}; do
  BENCH_NO_CPU=1 timeout ${TMO:-600} python bench.py --config $c --steps ${STEPS:-3} --warmup ${WARM:-1} > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "c$c rc=$?" >> gpurun_out/configs_rc.txt
done
