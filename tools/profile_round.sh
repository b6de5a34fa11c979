#!/usr/bin/env bash
# One GPU-box session that regenerates the measurement artefacts of a round (run from the repo root
# under gpurun; every ncu pass runs only after the same command exited 0 without ncu).
#   TAG=r01b bash tools/profile_round.sh
set -u
TAG=${TAG:-r01}
O=gpurun_out
mkdir -p $O
# 1. bench lines (default = c5p5 headline with CPU baseline + GMRES; the other configs with GMRES)
python bench.py > $O/${TAG}_bench_c5p5.log 2>&1 && tail -1 $O/${TAG}_bench_c5p5.log > $O/${TAG}_bench_c5p5.json
for c in c2 c3 c4 c5p2 c5p4; do
  python bench.py --config $c --steps 50 --no-cpu-baseline > $O/${TAG}_bench_$c.log 2>&1 && tail -1 $O/${TAG}_bench_$c.log > $O/${TAG}_bench_$c.json
done
python -m pytest tests -q -m gpu > $O/${TAG}_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
# 2. launch list of the timed steps of the default bench command (cold, serialised; shares only).
#    The plain run records its autotuned tilings in a cache that the ncu run replays, and the timed
#    region is bracketed by cudaProfilerStart/Stop (STIGA_PROFILE_RANGE=1).
export STIGA_TUNE_CACHE=/tmp/stiga_tune_${TAG}.txt
rm -f $STIGA_TUNE_CACHE
STIGA_PROFILE_RANGE=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gmres > $O/${TAG}_plain.log 2>&1 && \
  STIGA_PROFILE_RANGE=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file $O/${TAG}_launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gmres > $O/${TAG}_ncu_launches.log 2>&1
# 3. one apply per config, full set, per-launch raw page (same tuned tilings as the plain run)
for c in c5p5 c2 c3 c4; do
  python tools/profile_fd.py --config $c --names-out $O/${TAG}_names_$c.json > $O/${TAG}_pf_$c.log 2>&1 && \
  ncu --set full --clock-control none --profile-from-start off -o $O/${TAG}_$c \
      python tools/profile_fd.py --config $c > $O/${TAG}_ncu_$c.log 2>&1 && \
  ncu -i $O/${TAG}_$c.ncu-rep --page raw --csv > $O/${TAG}_${c}_raw.csv; rm -f $O/${TAG}_$c.ncu-rep
done
# 4. the system mat-vecs: c4 physical (stencil kernel + banded time pass), c3 Kronecker-sum form
for c in c4 c3; do
  python tools/profile_matvec.py --config $c > $O/${TAG}_pm_$c.log 2>&1 && \
  ncu --set full --clock-control none --profile-from-start off -o $O/${TAG}_matvec_$c \
      python tools/profile_matvec.py --config $c > $O/${TAG}_ncu_matvec_$c.log 2>&1 && \
  ncu -i $O/${TAG}_matvec_$c.ncu-rep --page raw --csv > $O/${TAG}_matvec_${c}_raw.csv; rm -f $O/${TAG}_matvec_$c.ncu-rep
done
ls -la $O | grep $TAG
