O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/dfma_probe tools/dfma_mode_probe.cu > $O/r03c_dfma_build.log 2>&1
timeout 600 /tmp/dfma_probe > $O/r03c_dfma.log 2>&1
for shp in "67 287496" "98 912672" "258 66048"; do
  tag=$(echo $shp | cut -d' ' -f1)
  timeout 900 ncu --set full --clock-control none -k regex:dfma_mode_kernel -c 12 -o $O/r03c_dfma_$tag /tmp/dfma_probe $shp > $O/r03c_ncu_dfma_$tag.log 2>&1 && \
  ncu -i $O/r03c_dfma_$tag.ncu-rep --page raw --csv > $O/r03c_dfma_${tag}_raw.csv; rm -f $O/r03c_dfma_$tag.ncu-rep
done
for c in c4 c3 c2; do
  STIGA_TIME_VARIANT=split python tools/profile_fd.py --config $c --names-out $O/r03c_names_${c}split.json > $O/r03c_pf_${c}split.log 2>&1 && \
  STIGA_TIME_VARIANT=split timeout 1500 ncu --set full --clock-control none --profile-from-start off -o $O/r03c_${c}split \
      python tools/profile_fd.py --config $c > $O/r03c_ncu_${c}split.log 2>&1 && \
  ncu -i $O/r03c_${c}split.ncu-rep --page raw --csv > $O/r03c_${c}split_raw.csv; rm -f $O/r03c_${c}split.ncu-rep
done
