# full GPU suite, smoke and bench line on the current tree (round 2, after the codepoint work)
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
echo done
