# usage: bash scripts/ncu_k1.sh <tag> [env assignments...]
tag=$1; shift
env "$@" ncu --set full --clock-control none --import-source on -k regex:k_signature -s 1 -c 1 -o gpurun_out/k1_$tag python scripts/probe_k1.py 200000 128 > gpurun_out/ncu_k1_$tag.log 2>&1
tail -3 gpurun_out/ncu_k1_$tag.log
