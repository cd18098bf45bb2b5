# quick GPU pass: selected tests (TESTS, default the exactness file) + A/B of variant libraries
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ -z "$NOTEST" ] && timeout 1500 python -m pytest ${TESTS:-tests/test_k3_exact.py} -x -q > gpurun_out/k3exact.log 2>&1; echo "rc=$?" >> gpurun_out/k3exact.log
for lib in ${VARIANTS:-paper_2504_14966_b200/libslosched_b200.so paper_2504_14966_b200/_variants/*.so}; do
  echo "== $lib"; SLOSCHED_LIB=$lib timeout 300 python tools/prof_chains.py --bench --reps 3 | tail -1
  SLOSCHED_LIB=$lib timeout 300 python tools/prof_chains.py --bench --reps 2 --n 4096 --levels 4 | tail -1
done > gpurun_out/ab.log 2>&1
tail -30 gpurun_out/k3exact.log; cat gpurun_out/ab.log
