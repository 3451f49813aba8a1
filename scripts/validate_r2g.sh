# final round-2 validation (after the budget-query cache and the 48 MB first chunk): full GPU suite, smoke, bench line, reference arm
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2g_bench_reference.json 2> gpurun_out/r2g_bench_reference.err
echo done
