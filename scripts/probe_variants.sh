# K1 throughput per library variant (device-resident 1M docs)
for v in "$@"; do
  echo "== $v"
  ND_LIB_PATH=build/variants/lib_$v.so python scripts/probe_k1.py 1000000 128 2>&1 | grep -E "iter 4|host=="
done
