for fz in 8,2 4,1 16,4; do echo "== FZ $fz"; ND_K1_FZ=$fz python scripts/probe_k1.py 1000000 128 2>&1 | grep -E "iter 4"; done
