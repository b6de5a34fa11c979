O=gpurun_out; mkdir -p $O
export STIGA_TUNE_CACHE=/tmp/stiga_tune_r03o.txt
rm -f $STIGA_TUNE_CACHE
python tools/profile_fd.py --config c4 --names-out $O/r03o_names_c4.json > $O/r03o_pf_c4.log 2>&1 && \
ncu --set full --import-source on --clock-control none --profile-from-start off -o $O/r03o_c4 \
    python tools/profile_fd.py --config c4 > $O/r03o_ncu_c4.log 2>&1 && \
ncu -i $O/r03o_c4.ncu-rep --page source --csv --print-source sass > $O/r03o_c4_src.csv
rm -f $O/r03o_c4.ncu-rep
