# Round-1 profiling pass (run under gpurun from the repo root)
set -x
python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
tail -3 gpurun_out/bench_r1b.err
# launch list of a short bench (device-timed K1 + e2e + dedup), cold-cache per launch
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
# full capture of K1 at the bench size (1M docs): first device-path launch after warm-up
ncu --set full --clock-control none --import-source on -k regex:k_signature -s 1 -c 1 -o gpurun_out/k1_full_1M python bench.py --steps 1 --warmup 1 --no-cpu --no-dedup > gpurun_out/ncu_k1_full.log 2>&1
# full capture of the compare kernel inside the 1M dedup
ncu --set full --clock-control none --import-source on -k regex:k_compare -c 1 -o gpurun_out/k3_full_1M python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_k3_full.log 2>&1
ls -la gpurun_out
