# quick GPU pass: selected tests (TESTS, default the exactness file) + A/B of variant libraries
# (fixed-work chain launches at the bench shape for each N in NS)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ -z "$NOTEST" ] && timeout 1500 python -m pytest ${TESTS:-tests/test_k3_exact.py} -x -q > gpurun_out/k3exact.log 2>&1; echo "rc=$?" >> gpurun_out/k3exact.log
for lib in ${VARIANTS:-paper_2504_14966_b200/libslosched_b200.so paper_2504_14966_b200/_variants/*.so}; do
  echo "== $lib"
  for n in ${NS:-1024 4096}; do
   for mb in ${MBS:-4}; do
    lv=8; [ "$n" -gt 1024 ] && lv=4
    echo -n "n=$n mb=$mb "; SLOSCHED_LIB=$lib timeout 300 python tools/prof_chains.py --bench --reps 2 --n $n --mb $mb --levels $lv | tail -1
   done
  done
done > gpurun_out/ab.log 2>&1
tail -30 gpurun_out/k3exact.log; cat gpurun_out/ab.log
