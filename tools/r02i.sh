O=gpurun_out; mkdir -p $O
export STIGA_TUNE_CACHE=/tmp/stiga_tune_r02i.txt
python tools/profile_fd.py --config c4 --names-out $O/r02i_names_c4.json > $O/r02i_pf.log 2>&1 && \
ncu --set full --import-source on --clock-control none --profile-from-start off \
    -o $O/r02i_c4 python tools/profile_fd.py --config c4 > $O/r02i_ncu.log 2>&1
ncu -i $O/r02i_c4.ncu-rep --page raw --csv > $O/r02i_c4_raw.csv 2>&1
for i in 0 3; do ncu -i $O/r02i_c4.ncu-rep --page source --csv --launch-skip $i --launch-count 1 > $O/r02i_c4_src_$i.csv 2>&1; done
rm -f $O/r02i_c4.ncu-rep
python tools/profile_matvec.py --config c4 > $O/r02i_pm.log 2>&1 && \
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:stencil \
    -o $O/r02i_mv python tools/profile_matvec.py --config c4 > $O/r02i_ncu_mv.log 2>&1
ncu -i $O/r02i_mv.ncu-rep --page raw --csv > $O/r02i_mv_raw.csv 2>&1
ncu -i $O/r02i_mv.ncu-rep --page source --csv > $O/r02i_mv_src.csv 2>&1
rm -f $O/r02i_mv.ncu-rep
