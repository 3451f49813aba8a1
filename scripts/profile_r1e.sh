# Round-1 profiling pass #3 (run under gpurun from the repo root): tests, bench,
# launch list, ncu of K1 and the block join, paper-scale configs
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_r1e.log 2>&1; echo rc=$? >> gpurun_out/gpu_r1e.log
python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r1e.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-staged > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/dedup_kernels_r1e.csv python scripts/dedup_once.py 1000000 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_signature -s 1 -c 1 -o gpurun_out/k1_full_r1e \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-dedup --no-staged > gpurun_out/ncu_k1_r1e.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_join -s 1 -c 1 -o gpurun_out/kjoin_full_r1e \
    python scripts/dedup_once.py 1000000 > gpurun_out/ncu_kjoin_r1e.log 2>&1
for c in c3 c4 c5; do timeout 900 python scripts/run_configs.py $c --sample 2000 --out gpurun_out/r1_config_${c}_e.json > gpurun_out/${c}_e.log 2>&1; done
