O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02a_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x > $O/r02a_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02a_smoke.log 2>&1
timeout 600 python bench.py > $O/r02a_bench.log 2>&1
timeout 300 python tools/time_matvec.py c3 c4 c5p5 > $O/r02a_matvec.log 2>&1
for c in c3 c4 c2; do timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > $O/r02a_bench_$c.log 2>&1; done
