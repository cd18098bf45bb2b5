# mb = 8 (the max batch SURVEY 8(a) lists beside 4): fixed-work timings, one ncu capture of
# k_chains<1> at N=1024 mb=8, and the bench line at mb=8; plus a small-N capture (N=24, the online
# driver's per-instance queues).
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 300 python tools/prof_chains.py --bench --reps 3 --mb 8 > gpurun_out/prof_mb8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 \
    -o gpurun_out/k_chains_mb8 python tools/prof_chains.py --bench --mb 8 > gpurun_out/ncu_mb8.log 2>&1
P=$(grep -o "^rep 0: [0-9]*" gpurun_out/prof_mb8.log | awk '{print $3}')
python tools/ncu_summary.py gpurun_out/k_chains_mb8.ncu-rep --proposals $P --tag $TAG --n 1024 --mb 8 \
    --out k_chains_summary_n1024_mb8.json --desc "k_chains<1> (N=1024, mb=8, 16384 chains, prof_chains.py --bench --mb 8)" \
    > /dev/null 2>&1 && cp profiles/$TAG/k_chains_summary_n1024_mb8.json gpurun_out/
timeout 600 python bench.py --mb 8 --steps 50 > gpurun_out/bench_mb8.json 2> gpurun_out/bench_mb8.err
timeout 300 python tools/prof_chains.py 24 4096 2 > gpurun_out/prof_n24.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 \
    -o gpurun_out/k_chains_n24 python tools/prof_chains.py 24 4096 1 > gpurun_out/ncu_n24.log 2>&1
cat gpurun_out/prof_mb8.log gpurun_out/prof_n24.log
