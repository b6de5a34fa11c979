O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_geometry.py -q -m gpu -x -k "line_pair" > $O/r03g_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03g_pytest.log
for pf in 4 2 8 16; do
  STIGA_STENCIL_PF=$pf timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03g_pm_c4_pf$pf.log 2>&1
done
STIGA_STENCIL_NO_PREFETCH=1 timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03g_pm_c4_nopf.log 2>&1
