ncu --set full --clock-control none --import-source on -k regex:k_compare -c 1 -o gpurun_out/k3_$1 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_k3_$1.log 2>&1
tail -2 gpurun_out/ncu_k3_$1.log
