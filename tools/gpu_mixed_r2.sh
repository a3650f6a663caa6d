# c4 mixed-precision line (fp32 + fp64 refinement of the floor problems) and the full-batch fp32 floor count
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
BENCH_NO_CPU=1 timeout 600 python bench.py --precision mixed --no-op-bench > gpurun_out/bench_c4_mixed.json 2> gpurun_out/bench_c4_mixed.err
timeout 900 python -m pytest tests/test_gpu_full.py -m gpu -q -s -k "c4_full_batch" > gpurun_out/c4_full.log 2>&1
cat gpurun_out/bench_c4_mixed.json; tail -30 gpurun_out/c4_full.log
