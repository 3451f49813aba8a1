set -x
for a in dn fq dn fq; do ND_K1J_ARITH=$a timeout 300 python scripts/probe_k1.py 1000000 128 2>&1 | grep -E "iter|host e2e|==" | sed "s/^/$a /"; done > gpurun_out/k1ab.txt
for a in dn fq; do ND_K1J_ARITH=$a timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1j -s 1 -c 1 -o gpurun_out/k1j_$a python scripts/probe_k1.py 1000000 128 > gpurun_out/ncu_k1j_$a.log 2>&1; done
echo ok
