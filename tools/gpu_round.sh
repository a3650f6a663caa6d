#!/bin/bash
# One gpurun call: GPU tests, default bench, launch list + one full ncu capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
export PROF_B=${PROF_B:-296}
timeout 300 python tools/prof_c4.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_c4.py > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_s_recover -c 1 -o gpurun_out/prof_c4 python tools/prof_c4.py > gpurun_out/ncu_full.log 2>&1
echo done
