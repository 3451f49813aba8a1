# final round-2 validation (after the ASCII fast path and the GC fix): full GPU suite, smoke, bench line, reference arm
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2f_bench_reference.json 2> gpurun_out/r2f_bench_reference.err
echo done
