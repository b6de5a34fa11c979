O=gpurun_out; mkdir -p $O
export STIGA_TUNE_CACHE=/tmp/stiga_tune_r02c.txt
python tools/profile_fd.py --config c5p5 --names-out $O/r02c_names_c5p5.json > $O/r02c_pf.log 2>&1 && \
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:'fold|mode_product|scale|arrow' -c 11 \
    -o $O/r02c_c5p5 python tools/profile_fd.py --config c5p5 > $O/r02c_ncu.log 2>&1
ncu -i $O/r02c_c5p5.ncu-rep --page raw --csv > $O/r02c_c5p5_raw.csv 2>&1
for i in 1 4 9; do ncu -i $O/r02c_c5p5.ncu-rep --page source --csv --launch-skip $i --launch-count 1 > $O/r02c_c5p5_src_$i.csv 2>&1; done
ls -la $O | grep r02c
rm -f $O/r02c_c5p5.ncu-rep
