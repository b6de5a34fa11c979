O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_system_gpu.py -q -m gpu -x > $O/r02u_pytest.log 2>&1
timeout 300 python tools/time_matvec.py c3 c5p5 c2 c5p4 > $O/r02u_matvec.log 2>&1
python tools/profile_matvec.py --config c3 > $O/r02u_pm.log 2>&1 && \
ncu --set full --clock-control none --profile-from-start off -o $O/r02u_mv python tools/profile_matvec.py --config c3 > $O/r02u_ncu.log 2>&1
ncu -i $O/r02u_mv.ncu-rep --page raw --csv > $O/r02u_mv_raw.csv 2>&1
ncu -i $O/r02u_mv.ncu-rep --page source --csv --launch-skip 1 --launch-count 1 > $O/r02u_mv_src_stream.csv 2>&1
ncu -i $O/r02u_mv.ncu-rep --page source --csv --launch-skip 0 --launch-count 1 > $O/r02u_mv_src_plane.csv 2>&1
rm -f $O/r02u_mv.ncu-rep
