# Profile pass (B200 via gpurun): fixed-work timings + one ncu --set full capture of k_chains at the
# bench shape (N=1024) and at configs[3]'s shard (N=4096), summaries into gpurun_out/.
#   gpurun --timeout 1800 -- 'bash tools/gpu_prof.sh'
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 300 python tools/prof_chains.py --bench --reps 3 > gpurun_out/prof_chains.log 2>&1
timeout 300 python tools/prof_chains.py --bench --reps 2 --n 4096 --levels 4 >> gpurun_out/prof_chains.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 \
    -o gpurun_out/k_chains python tools/prof_chains.py --bench > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/k_chains.ncu-rep --proposals 39321600 --tag $TAG > /dev/null 2>&1 && \
    cp profiles/$TAG/k_chains_summary.json gpurun_out/k_chains_summary.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 \
    -o gpurun_out/k_chains_n4096 python tools/prof_chains.py --bench --n 4096 --levels 4 > gpurun_out/ncu_full_n4096.log 2>&1
python tools/ncu_summary.py gpurun_out/k_chains_n4096.ncu-rep --proposals 19660800 --tag $TAG --n 4096 --mb 4 \
    --out k_chains_summary_n4096_mb4.json --desc "k_chains<4> (N=4096, mb=4, 16384 chains, prof_chains.py --bench --n 4096 --levels 4)" \
    > /dev/null 2>&1 && cp profiles/$TAG/k_chains_summary_n4096_mb4.json gpurun_out/
[ -n "$BENCH" ] && timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/prof_chains.log
