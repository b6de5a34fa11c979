O=gpurun_out; mkdir -p $O
for c in c3 c2 c5p4; do
  STIGA_MATVEC_CONST=1 timeout 900 python tools/time_matvec.py $c > $O/r03i_tm_${c}_const.log 2>&1
  timeout 900 python tools/time_matvec.py $c > $O/r03i_tm_${c}_smem.log 2>&1
done
STIGA_MATVEC_CONST=1 timeout 900 python -m pytest tests/test_system_gpu.py -q -m gpu -x > $O/r03i_pytest_const.log 2>&1; echo "rc=$?" >> $O/r03i_pytest_const.log
for c in c2 c5p4; do
  timeout 900 python bench.py --config $c --steps 30 --no-cpu-baseline --no-gmres > $O/r03i_bench_${c}_base.log 2>&1
  STIGA_ARROW_PERSISTENT=1 timeout 900 python bench.py --config $c --steps 30 --no-cpu-baseline --no-gmres > $O/r03i_bench_${c}_pers.log 2>&1
done
STIGA_ARROW_PERSISTENT=1 timeout 900 python -m pytest tests/test_fd_gpu.py -q -m gpu -x -k "time_variants or c2 or nt1" > $O/r03i_pytest_pers.log 2>&1; echo "rc=$?" >> $O/r03i_pytest_pers.log
