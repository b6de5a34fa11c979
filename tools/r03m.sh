O=gpurun_out; mkdir -p $O
TAG=r03x
timeout 1500 python -m pytest tests/test_geometry.py tests/test_system_gpu.py tests/test_distributed_gpu.py -q -m gpu -x > $O/r03m_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03m_pytest.log
python bench.py --config c4 --steps 50 --no-cpu-baseline > $O/${TAG}_bench_c4.log 2>&1 && tail -1 $O/${TAG}_bench_c4.log > $O/${TAG}_bench_c4.json
STIGA_STENCIL_NO_PAIR=1 timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03m_pm_c4_old.log 2>&1
for c in c4; do
  python tools/profile_matvec.py --config $c > $O/${TAG}_pm_$c.log 2>&1 && \
  ncu --set full --import-source on --clock-control none --profile-from-start off -o $O/${TAG}_matvec_$c \
      python tools/profile_matvec.py --config $c > $O/${TAG}_ncu_matvec_$c.log 2>&1 && \
  ncu -i $O/${TAG}_matvec_$c.ncu-rep --page raw --csv > $O/${TAG}_matvec_${c}_raw.csv && \
  ncu -i $O/${TAG}_matvec_$c.ncu-rep --page source --csv --print-source sass > $O/r03m_matvec_${c}_src.csv
  rm -f $O/${TAG}_matvec_$c.ncu-rep
done
python -c "import __graft_entry__ as g; g.smoke()" > $O/r03m_smoke.log 2>&1
