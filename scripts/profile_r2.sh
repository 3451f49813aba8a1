# Round-2 measurement pass (run under gpurun from the repo root): launch lists
# of the bench and of one C2 dedup, ncu --set full of K1j at the bench size
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-staged --no-c3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r2_dedup_kernels_1M.csv python scripts/dedup_once.py 1000000 > /dev/null 2>&1
ncu --kernel-name regex:"k1j" --launch-skip 1 --launch-count 1 --set full --import-source on \
    -o gpurun_out/r2_k1j_full_1M python scripts/k1_probe_once.py 1000000 > gpurun_out/r2_k1j_ncu.log 2>&1
ncu --kernel-name regex:"k_join_blocks" --launch-skip 1 --launch-count 1 --set full \
    -o gpurun_out/r2_kjoin_full_1M python scripts/dedup_once.py 1000000 > gpurun_out/r2_kjoin_ncu.log 2>&1
echo done
