#!/bin/bash
# Round measurement: GPU tests, default bench (c4, with the CPU baseline), the other configs,
# the c4 launch list, full ncu captures of the c4 and c5 recovery kernels.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
for c in 1 2 3 5; do
  BENCH_NO_CPU=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
BENCH_NO_CPU=1 timeout 600 python bench.py --config 4 --alg cosamp --steps 5 --warmup 3 > gpurun_out/bench_c4_cosamp.json 2> gpurun_out/bench_c4_cosamp.err
BENCH_NO_CPU=1 timeout 600 python bench.py --config 4 --randomizer perm --steps 5 --warmup 3 > gpurun_out/bench_c4_perm.json 2> gpurun_out/bench_c4_perm.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
export PROF_B=4096
timeout 300 python tools/prof_c4.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_c4.py > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_s_recover -c 1 -o gpurun_out/prof_c4 python tools/prof_c4.py > gpurun_out/ncu_full.log 2>&1
export PROF_CFG=5
timeout 300 python tools/prof_cfg.py > gpurun_out/prof_plain5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_l_recover -c 1 -o gpurun_out/prof_c5 python tools/prof_cfg.py > gpurun_out/ncu_full5.log 2>&1
# summaries here on the box; the reports themselves stay off gpurun_out (64 MiB cap)
mkdir -p /tmp/ncu && mv gpurun_out/*.ncu-rep /tmp/ncu/ 2>/dev/null
for r in prof_c4 prof_c5; do
  [ -f /tmp/ncu/$r.ncu-rep ] && python tools/ncu_summary.py /tmp/ncu/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1
done
export TRAFFIC_JSON=gpurun_out/traffic.json
[ -f /tmp/ncu/prof_c4.ncu-rep ] && python tools/traffic_from_ncu.py /tmp/ncu/prof_c4.ncu-rep c4_fp32 k_s_recover
[ -f /tmp/ncu/prof_c5.ncu-rep ] && python tools/traffic_from_ncu.py /tmp/ncu/prof_c5.ncu-rep c5_fp32 k_l_recover
# keep the c4 report if it is small enough to travel
[ -f /tmp/ncu/prof_c4.ncu-rep ] && [ $(stat -c %s /tmp/ncu/prof_c4.ncu-rep) -lt 40000000 ] && cp /tmp/ncu/prof_c4.ncu-rep gpurun_out/
echo done
