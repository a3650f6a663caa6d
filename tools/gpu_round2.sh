#!/bin/bash
# Round-2 evidence with the final build: launch list of the bench command (c4), full ncu captures of
# the c4 (full 4096 batch) and c5 recovery kernels, summaries + per-line exports, traffic.json.
mkdir -p gpurun_out /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-op-bench > gpurun_out/ncu_launch.log 2>&1
export PROF_B=4096
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_s_recover -c 1 -o /tmp/ncu/c4_full python tools/prof_c4.py > gpurun_out/ncu_c4.log 2>&1
export PROF_CFG=5
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_l_recover -c 1 -o /tmp/ncu/c5_full python tools/prof_cfg.py > gpurun_out/ncu_c5.log 2>&1
export PROF_CFG=3
timeout 1500 ncu --set full --clock-control none -k regex:k_l_recover -c 1 -o /tmp/ncu/c3_full python tools/prof_cfg.py > gpurun_out/ncu_c3.log 2>&1
for r in c4_full c5_full c3_full; do
  [ -f /tmp/ncu/$r.ncu-rep ] && bash tools/ncu_export.sh /tmp/ncu/$r.ncu-rep gpurun_out/$r
done
export TRAFFIC_JSON=gpurun_out/traffic.json
cp profiles/traffic.json gpurun_out/traffic.json
[ -f /tmp/ncu/c4_full.ncu-rep ] && python tools/traffic_from_ncu.py /tmp/ncu/c4_full.ncu-rep c4_fp32 k_s_recover
[ -f /tmp/ncu/c5_full.ncu-rep ] && python tools/traffic_from_ncu.py /tmp/ncu/c5_full.ncu-rep c5_fp32 k_l_recover
[ -f /tmp/ncu/c3_full.ncu-rep ] && python tools/traffic_from_ncu.py /tmp/ncu/c3_full.ncu-rep c3_fp32 k_l_recover
ls -la gpurun_out
