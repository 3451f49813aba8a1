# Round-1 profiling pass #2 (run under gpurun from the repo root)
python bench.py > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err
# every kernel of one in-memory dedup (C2, 1M docs): duration + DRAM bytes per launch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/dedup_kernels_r1c.csv python scripts/dedup_once.py 1000000 > gpurun_out/dedup_once.log 2>&1
python scripts/ncu_launch_summary.py gpurun_out/dedup_kernels_r1c.csv > gpurun_out/dedup_kernels_r1c.txt 2>&1
# full capture of K1 at the bench size with source and stall reasons
ncu --set full --clock-control none --import-source on -k regex:k_signature -s 1 -c 1 -o gpurun_out/k1_full_r1c \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-dedup > gpurun_out/ncu_k1_r1c.log 2>&1
# full capture of the hash-join compare kernel inside the 1M dedup
ncu --set full --clock-control none --import-source on -k regex:k_join -s 1 -c 1 -o gpurun_out/kjoin_full_r1c \
    python scripts/dedup_once.py 1000000 > gpurun_out/ncu_kjoin_r1c.log 2>&1
ls -la gpurun_out
