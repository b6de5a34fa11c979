O=gpurun_out; mkdir -p $O
for c in c4 c5p2 c3 c2 c5p4; do
  timeout 900 python bench.py --config $c --steps 50 --no-cpu-baseline --no-gmres > $O/r03p_bench_$c.log 2>&1
done
timeout 2400 python -m pytest tests/test_fd_gpu.py tests/test_distributed_gpu.py -q -m gpu -x > $O/r03p_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03p_pytest.log
