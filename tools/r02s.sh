O=gpurun_out; mkdir -p $O
for c in c5p5 c3; do
STIGA_DEBUG_TUNE=1 timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline --no-gmres > $O/r02s_bench_$c.log 2>&1
done
