# K3 time on the bench shard at C2 (K=2000, ~500-document cells) and C3-like
# (K=365, ~2740-document cells) cell sizes, H=128 and 256; $1 = env settings to compare
for E in "${@:-X=1}"; do for K in 365 2000; do for H in 128 256; do
  echo -n "$E K=$K H=$H "; env $E python scripts/dedup_once.py 1000000 $H $K | python -c "import sys,ast; l=sys.stdin.read(); s=ast.literal_eval(l[l.index('['):]); print('pairs', l.split()[4], 'K3 %.2f ms' % (s[2]*1e3))"
done; done; done
