O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_geometry.py tests/test_system_gpu.py tests/test_setup_device.py -q -m gpu -x > $O/r02w_pytest.log 2>&1
timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r02w_pm_c4.log 2>&1
timeout 600 python bench.py --config c4 --steps 30 --no-cpu-baseline > $O/r02w_bench_c4.log 2>&1
