#!/bin/bash
# One full ncu capture of the top Tier S kernel on a one-wave c4 batch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export PROF_B=${PROF_B:-148}
timeout 300 python tools/prof_c4.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_s_recover} -c 1 -o gpurun_out/${PROF_NAME:-prof_c4} python tools/prof_c4.py > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
