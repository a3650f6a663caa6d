# host-buffer pipeline with refine_fp64: new parity test, every host-path test, mixed + default bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_extras.py tests/test_gpu_recover.py -m gpu -q -x -k "host or refine" > gpurun_out/refine_host.log 2>&1; echo "pytest rc=$?" >> gpurun_out/refine_host.log
BENCH_NO_CPU=1 timeout 600 python bench.py --precision mixed --no-op-bench > gpurun_out/bench_c4_mixed.json 2> gpurun_out/bench_c4_mixed.err
tail -5 gpurun_out/refine_host.log; cat gpurun_out/bench_c4_mixed.json; tail -3 gpurun_out/bench_c4_mixed.err
