#!/bin/bash
# Final round-2 evidence with the final build: the c4 bench launch list, full ncu captures of the
# c5 and c3 grid-tier recoveries (summaries, per-line exports, traffic), then every bench line.
mkdir -p gpurun_out /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-op-bench > gpurun_out/ncu_launch.log 2>&1
export TRAFFIC_JSON=gpurun_out/traffic.json
cp profiles/traffic.json gpurun_out/traffic.json
for cfg in 5 3; do
  PROF_CFG=$cfg timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_l_recover -c 1 \
    -o /tmp/ncu/c${cfg}_full python tools/prof_cfg.py > gpurun_out/ncu_c$cfg.log 2>&1
  [ -f /tmp/ncu/c${cfg}_full.ncu-rep ] && bash tools/ncu_export.sh /tmp/ncu/c${cfg}_full.ncu-rep gpurun_out/c${cfg}_full \
    && python tools/traffic_from_ncu.py /tmp/ncu/c${cfg}_full.ncu-rep c${cfg}_fp32 k_l_recover
done
bash tools/gpu_bench_all.sh > gpurun_out/bench_all.log 2>&1
