O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_setup_device.py tests/test_spacetime_system.py -q -m gpu > $O/r02h_pytest_setup.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $O/r02h_pytest_gpu.log 2>&1
