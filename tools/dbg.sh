set -x
for t in "test_best_exchange_vs_oracle_sizes" "test_best_exchange_near_ties_and_converged"; do
  for m in None fp64 filter32; do
    timeout 120 python -m pytest "tests/test_gpu_parity.py::${t}[${m}]" -x -q --timeout 100 > gpurun_out/dbg_${t}_${m}.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_${t}_${m}.log
  done
done
timeout 200 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
