O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_geometry.py -q -m gpu -x -k "line_pair or physical_system" > $O/r03k_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03k_pytest.log
timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03k_pm_c4.log 2>&1
timeout 600 python bench.py --config c4 --steps 30 --no-cpu-baseline > $O/r03k_bench_c4.log 2>&1
