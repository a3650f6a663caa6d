mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g4_pytest.log
for c in 2 3 5; do BENCH_NO_CPU=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/g4_bench_c$c.json 2> gpurun_out/g4_bench_c$c.err; done
