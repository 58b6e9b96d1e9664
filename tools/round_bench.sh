# Round-end measurements on one B200 (run through gpurun from the repo
# root): every bench config's line, the reference arm, the C2 launch list,
# ncu --set full of the dominant kernel at C2 and C3.  Outputs under
# gpurun_out/; the summaries worth keeping are copied to profiles/<round>/.
#   bash tools/round_bench.sh [configs...]
set -u
mkdir -p gpurun_out
CONFIGS=${*:-"c2 c2i c2s c1 c3 c3s c4 c5"}
for c in $CONFIGS; do
  steps=200; [ $c = c4 ] && steps=10; [ $c = c5 ] && steps=10
  [ $c = c3 ] && steps=50; [ $c = c3s ] && steps=50
  timeout 900 python bench.py --config $c --steps $steps --warmup 5 \
    > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$? $(tail -c 300 gpurun_out/bench_$c.json)"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 \
  > gpurun_out/reference_arm_c2.json 2> gpurun_out/reference_arm_c2.err
echo "reference rc=$?"
