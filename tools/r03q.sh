O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/r03q_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r03q_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r03q_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r03q_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/r03q_bench_ref.log 2>&1
timeout 900 python bench.py > $O/r03q_bench_default.log 2>&1
