# usage: bash scripts/ncu_kernel.sh <kernel-regex> <tag> [bench args]
k=$1; tag=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/$tag python bench.py --steps 1 --warmup 1 --no-cpu "$@" > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
