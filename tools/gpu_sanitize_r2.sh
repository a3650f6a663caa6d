#!/bin/bash
# compute-sanitizer over small recoveries on every tier / algorithm / precision (tools/sanitize_small.py):
# memcheck (out-of-bounds / misaligned global and shared accesses), racecheck (shared-memory hazards),
# synccheck (illegal barrier use). Each bounded by its own timeout.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.log
timeout 1200 $CS --tool racecheck --racecheck-report analysis --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
for f in gpurun_out/san_*.log; do echo "== $f"; tail -4 $f; done
