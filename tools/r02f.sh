O=gpurun_out; mkdir -p $O
export STIGA_FOLD_KERNEL=res
python tools/profile_fd.py --config c3 --names-out $O/r02f_names.json > $O/r02f_pf.log 2>&1 && \
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'fold' -c 4 \
    -o $O/r02f_c3 python tools/profile_fd.py --config c3 > $O/r02f_ncu.log 2>&1
ncu -i $O/r02f_c3.ncu-rep --page raw --csv > $O/r02f_c3_raw.csv 2>&1
for i in 0 1; do ncu -i $O/r02f_c3.ncu-rep --page source --csv --launch-skip $i --launch-count 1 > $O/r02f_c3_src_$i.csv 2>&1; done
rm -f $O/r02f_c3.ncu-rep
