O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_system_gpu.py tests/test_distributed_gpu.py -q -m gpu -x > $O/r02t_pytest.log 2>&1
timeout 300 python tools/time_matvec.py c3 c5p5 c2 > $O/r02t_matvec.log 2>&1
STIGA_PLANE2_SINGLE=1 timeout 300 python tools/time_matvec.py c3 c5p5 c2 > $O/r02t_matvec_single.log 2>&1
