# Round-1 final pass (run under gpurun from the repo root): smoke, tests, bench,
# launch lists of the bench and of one C2 dedup (K1..K4 after the K3 changes)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1f.log 2>&1; echo rc=$? >> gpurun_out/smoke_r1f.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_r1f.log 2>&1; echo rc=$? >> gpurun_out/gpu_r1f.log
python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-staged > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/dedup_kernels_r1f.csv python scripts/dedup_once.py 1000000 > /dev/null 2>&1
