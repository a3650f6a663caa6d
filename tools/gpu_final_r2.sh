#!/bin/bash
# Round-2 closing evidence with the final build: GPU tests, every bench line, the standalone
# operator / top-K table with its ncu summary, full ncu captures of the c5 and c3 recoveries
# (summaries, SASS exports, DRAM traffic), and the c4 bench launch list.
mkdir -p gpurun_out /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/gpu_bench_all.sh > gpurun_out/bench_all.log 2>&1
python tools/prof_ops.py > gpurun_out/ops_standalone.md 2> gpurun_out/ops.err
PROF_ONCE=1 timeout 900 ncu -f --set full --clock-control none -k regex:"k_s_apply|k_s_adjoint|k_l_apply|k_l_adjoint|k_l_diag_topk|k_s_diag_topk" \
  -o /tmp/ncu/ops python tools/prof_ops.py > gpurun_out/ncu_ops.log 2>&1
python tools/ncu_summary.py /tmp/ncu/ops.ncu-rep > gpurun_out/ncu_ops.txt 2>&1
export TRAFFIC_JSON=gpurun_out/traffic.json
cp profiles/traffic.json gpurun_out/traffic.json
for cfg in 5 3; do
  PROF_CFG=$cfg timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:k_l_recover -c 1 \
    -o /tmp/ncu/c${cfg}_full python tools/prof_cfg.py > gpurun_out/ncu_c$cfg.log 2>&1
  [ -f /tmp/ncu/c${cfg}_full.ncu-rep ] && bash tools/ncu_export.sh /tmp/ncu/c${cfg}_full.ncu-rep gpurun_out/c${cfg}_full \
    && python tools/traffic_from_ncu.py /tmp/ncu/c${cfg}_full.ncu-rep c${cfg}_fp32 k_l_recover
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --steps 2 --warmup 1 --no-op-bench > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
