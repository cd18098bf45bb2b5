# One GPU verification + measurement pass (run on a B200 box from the repo root, e.g.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh'
# ); outputs land in gpurun_out/. The summaries committed under profiles/<round>/ come from these
# files: python tools/ncu_summary.py gpurun_out/k_chains.ncu-rep --proposals <printed> --tag <round>
#   --launches gpurun_out/launches.csv
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
# fixed-work capture of the chain kernel in the bench configuration (prints the proposal count)
timeout 300 python tools/prof_chains.py --bench --reps 3 > gpurun_out/prof_chains.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 \
    -o gpurun_out/k_chains python tools/prof_chains.py --bench > gpurun_out/ncu_full.log 2>&1
# the bench's roofline reads profiles/${TAG:-r2}/k_chains_summary.json: refresh it from this capture
# (prof_chains.py --bench evaluates 16384 chains x 8 levels x 300 proposals = 39321600)
python tools/ncu_summary.py gpurun_out/k_chains.ncu-rep --proposals 39321600 --tag ${TAG:-r2} > /dev/null 2>&1 && \
    cp profiles/${TAG:-r2}/k_chains_summary.json gpurun_out/k_chains_summary.json
# the same for configs[3]'s shard (N=4096: k_chains<4>; 4 levels ~ what its 7.9 ms device budget allows)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 \
    -o gpurun_out/k_chains_n4096 python tools/prof_chains.py --bench --n 4096 --levels 4 > gpurun_out/ncu_full_n4096.log 2>&1
python tools/ncu_summary.py gpurun_out/k_chains_n4096.ncu-rep --proposals 19660800 --tag ${TAG:-r2} --n 4096 --mb 4 \
    --out k_chains_summary_n4096_mb4.json --desc "k_chains<4> (N=4096, mb=4, 16384 chains, prof_chains.py --bench --n 4096 --levels 4)" \
    > /dev/null 2>&1 && cp profiles/${TAG:-r2}/k_chains_summary_n4096_mb4.json gpurun_out/
# launch list of the bench command (times are cold-cache and serialised: use the shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > gpurun_out/b_ncu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --n 4096 > gpurun_out/bench_n4096.json 2> gpurun_out/bench_n4096.err
timeout 600 python bench.py --mb 8 > gpurun_out/bench_mb8.json 2> gpurun_out/bench_mb8.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 \
    -o gpurun_out/k_chains_mb8 python tools/prof_chains.py --bench --mb 8 > gpurun_out/ncu_mb8.log 2>&1
python tools/ncu_summary.py gpurun_out/k_chains_mb8.ncu-rep --proposals 39321600 --tag ${TAG:-r2} --n 1024 --mb 8 \
    --out k_chains_summary_n1024_mb8.json --desc "k_chains<1> (N=1024, mb=8, 16384 chains, prof_chains.py --bench --mb 8)" \
    > /dev/null 2>&1 && cp profiles/${TAG:-r2}/k_chains_summary_n1024_mb8.json gpurun_out/
# the short-queue kernel (K5) at an online window's shape (n=6: 384 chains x 10 levels x 30 = 115200)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chains_small -c 1 \
    -o gpurun_out/k5_n6 python tools/prof_small.py 6 > gpurun_out/ncu_k5.log 2>&1
python tools/ncu_summary.py gpurun_out/k5_n6.ncu-rep --proposals 115200 --tag ${TAG:-r2} --n 6 --mb 4 \
    --out k5_summary_n6.json --desc "k_chains_small (N=6, mb=4, 384 chains, tools/prof_small.py 6)" \
    > /dev/null 2>&1 && cp profiles/${TAG:-r2}/k5_summary_n6.json gpurun_out/
[ -n "$ONLINE" ] && timeout 1500 python tools/online_bench.py --n 100000 --policies sa,fcfs,ref \
    --out gpurun_out/online_config5.json > gpurun_out/online.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/san_$t.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/prof_chains.log gpurun_out/bench.json
