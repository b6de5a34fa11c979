O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_fd_gpu.py -q -m gpu -x -k "time_resident or time_variants" > $O/r02r_pytest.log 2>&1
