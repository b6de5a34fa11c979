O=gpurun_out; mkdir -p $O
TAG=r03x
timeout 1500 python -m pytest tests/test_geometry.py tests/test_system_gpu.py tests/test_spacetime_system.py -q -m gpu -x > $O/r03n_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03n_pytest.log
STIGA_STENCIL_NO_TIME_FUSION=1 timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03n_pm_c4_unfused.log 2>&1
timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03n_pm_c4_fused.log 2>&1
python bench.py --config c4 --steps 50 --no-cpu-baseline > $O/r03n_bench_c4.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/r03n_smoke.log 2>&1
