O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_fd_gpu.py -q -m gpu -x -k "time_resident or time_variants" > $O/r02q_pytest.log 2>&1
for c in c4 c5p2 c3; do
STIGA_DEBUG_TUNE=1 timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline --no-gmres > $O/r02q_bench_$c.log 2>&1
done
