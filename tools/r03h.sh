O=gpurun_out; mkdir -p $O
for c in c3 c2 c5p4; do
  timeout 900 python tools/time_matvec.py $c > $O/r03h_tm_${c}_lds.log 2>&1
  STIGA_MATVEC_LDGC=1 timeout 900 python tools/time_matvec.py $c > $O/r03h_tm_${c}_ldg.log 2>&1
done
timeout 600 python tools/profile_matvec.py --config c4 --applies 3 > $O/r03h_pm_c4.log 2>&1
