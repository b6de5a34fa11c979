#!/usr/bin/env bash
# One GPU-box session that regenerates the measurement artefacts of a round (run from the repo root
# under gpurun; every ncu pass runs only after the same command exited 0 without ncu).
#   TAG=r01b bash tools/profile_round.sh
set -u
TAG=${TAG:-r01}
O=gpurun_out
mkdir -p $O
# 1. bench lines (default = c2 headline with CPU baseline + GMRES; c3, c4 with GMRES)
python bench.py > $O/${TAG}_bench_c2.log 2>&1 && tail -1 $O/${TAG}_bench_c2.log > $O/${TAG}_bench_c2.json
for c in c3 c4; do
  python bench.py --config $c --steps 100 --no-cpu-baseline > $O/${TAG}_bench_$c.log 2>&1 && tail -1 $O/${TAG}_bench_$c.log > $O/${TAG}_bench_$c.json
done
# 2. launch list of the default bench command (cold, serialised; shares only)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > $O/${TAG}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gmres > $O/${TAG}_ncu_launches.log 2>&1
# 3. one apply per config, full set, per-launch raw page
for c in c2 c3 c4; do
  python tools/profile_fd.py --config $c --names-out $O/${TAG}_names_$c.json > $O/${TAG}_pf_$c.log 2>&1 && \
  ncu --set full --clock-control none --profile-from-start off -o $O/${TAG}_$c \
      python tools/profile_fd.py --config $c > $O/${TAG}_ncu_$c.log 2>&1 && \
  ncu -i $O/${TAG}_$c.ncu-rep --page raw --csv > $O/${TAG}_${c}_raw.csv && rm -f $O/${TAG}_$c.ncu-rep
done
# 4. the physical mat-vec of c4 (stencil kernel + banded time pass)
python tools/profile_matvec.py > $O/${TAG}_pm.log 2>&1 && \
  ncu --set full --clock-control none --profile-from-start off -o $O/${TAG}_matvec \
      python tools/profile_matvec.py > $O/${TAG}_ncu_matvec.log 2>&1 && \
  ncu -i $O/${TAG}_matvec.ncu-rep --page raw --csv > $O/${TAG}_matvec_raw.csv && rm -f $O/${TAG}_matvec.ncu-rep
ls -la $O | grep $TAG
