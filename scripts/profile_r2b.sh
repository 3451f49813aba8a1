# Round-2 (second half) measurement pass under gpurun from the repo root:
# full GPU suite, smoke, bench line, launch lists of the bench and of one C2
# dedup, ncu --set full of K1j (dn arithmetic, F=32) at the bench size
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r2b_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-staged --no-c3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r2b_dedup_kernels_1M.csv python scripts/dedup_once.py 1000000 > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:"k1j" --launch-skip 1 --launch-count 1 --set full --clock-control none --import-source on \
    -o gpurun_out/r2b_k1j_full_1M python scripts/k1_probe_once.py 1000000 > gpurun_out/r2b_k1j_ncu.log 2>&1
echo done
