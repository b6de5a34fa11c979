O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_fd_gpu.py tests/test_distributed_gpu.py -q -m gpu -x > $O/r02n_pytest.log 2>&1
for c in c4 c3 c5p5 c2; do
STIGA_DEBUG_TUNE=1 timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline --no-gmres > $O/r02n_bench_$c.log 2>&1
done
