# ncu evidence for the round (one GPU, after the plain runs exit 0):
# the C2 launch list (cold-cache, serialised: compare shares) and
# --set full captures of the bounded 2-opt scan at C2 and C3, the update
# kernel at C2, and the band scan (DPSO_BOUND=0) at C2.
#   bash tools/round_ncu.sh <tag>
set -u
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/launches_${tag}_c2.csv \
  python bench.py --steps 3 --warmup 3 --profile-gens 2 --no-cpu-baseline \
  --no-e2e > gpurun_out/ncu_launch_${tag}.log 2>&1
echo "launch list rc=$?"
for c in c2 c3; do
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:k_two_opt_bound -s 8 -c 1 -o gpurun_out/bound_${tag}_$c -f \
    python bench.py --config $c --steps 12 --warmup 3 --profile-gens 1 \
    --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${tag}_$c.log 2>&1
  echo "ncu full bound $c rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_update_w1 -s 2 -c 1 -o gpurun_out/update_${tag}_c2 -f \
  python bench.py --config c2 --steps 3 --warmup 3 --profile-gens 1 \
  --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${tag}_upd.log 2>&1
echo "ncu full update c2 rc=$?"
DPSO_BOUND=0 timeout 900 ncu --set full --clock-control none \
  --import-source on -k regex:k_two_opt_band -s 2 -c 1 \
  -o gpurun_out/band_${tag}_c2 -f python bench.py --config c2 --steps 3 \
  --warmup 3 --profile-gens 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full_${tag}_band.log 2>&1
echo "ncu full band c2 rc=$?"
