O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_fd_gpu.py -q -m gpu -x -k "three_warp_rows or time_variants or full_baseline" > $O/r03b_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03b_pytest.log
for c in c4 c5p2 c5p4 c5p5; do
  STIGA_DEBUG_TUNE=1 timeout 900 python bench.py --config $c --steps 30 --no-cpu-baseline --no-gmres > $O/r03b_tune_$c.log 2>&1
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/dfma_probe tools/dfma_mode_probe.cu > $O/r03b_dfma_build.log 2>&1
timeout 600 /tmp/dfma_probe > $O/r03b_dfma.log 2>&1
