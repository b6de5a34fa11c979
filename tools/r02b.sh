O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_spacetime_system.py -q -m gpu -x > $O/r02b_pytest_system.log 2>&1
