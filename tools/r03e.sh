O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_geometry.py -q -m gpu -x -k "line_pair or tiling_edges or physical_system" > $O/r03e_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03e_pytest.log
timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03e_pm_c4_pair.log 2>&1
STIGA_STENCIL_NO_PAIR=1 timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03e_pm_c4_old.log 2>&1
timeout 600 python bench.py --config c4 --steps 30 --no-cpu-baseline > $O/r03e_bench_c4.log 2>&1
timeout 1500 python -m pytest tests/test_system_gpu.py tests/test_spacetime_system.py -q -m gpu -x > $O/r03e_pytest2.log 2>&1; echo "pytest rc=$?" >> $O/r03e_pytest2.log
