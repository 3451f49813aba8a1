# final round-2 validation: full GPU suite, smoke, bench line, reference arm
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2d_bench_reference.json 2> gpurun_out/r2d_bench_reference.err
echo done
