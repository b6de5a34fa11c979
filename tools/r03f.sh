O=gpurun_out; mkdir -p $O
for c in c4; do
  python tools/profile_matvec.py --config $c > $O/r03f_pm_$c.log 2>&1 && \
  timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -o $O/r03f_matvec_$c \
      python tools/profile_matvec.py --config $c > $O/r03f_ncu_matvec_$c.log 2>&1 && \
  ncu -i $O/r03f_matvec_$c.ncu-rep --page raw --csv > $O/r03f_matvec_${c}_raw.csv && \
  ncu -i $O/r03f_matvec_$c.ncu-rep --page source --csv --print-source sass > $O/r03f_matvec_${c}_src.csv
  rm -f $O/r03f_matvec_$c.ncu-rep
done
