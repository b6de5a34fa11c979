O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -x > $O/r03a_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r03a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r03a_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r03a_smoke.log
for c in c4 c5p2 c3; do
  STIGA_DEBUG_TUNE=1 timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline --no-gmres > $O/r03a_tune_$c.log 2>&1
done
timeout 900 python bench.py > $O/r03a_bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/r03a_bench_ref.log 2>&1
