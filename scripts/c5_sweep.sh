# K3 on C5 (clusters of 2-20: handled-pair set overflows) and the k3_sweep shapes
for E in "${@:-X=1}"; do
  env $E timeout 600 python scripts/run_configs.py c5 --sample 10 --out /tmp/c5.json > /dev/null 2>&1
  python -c "import json;d=json.load(open('/tmp/c5.json'));print('$E c5', d['dedup_ms'], 'K3', d['stage_seconds'][2], d['distinct_pairs'])"
done
bash scripts/k3_sweep.sh "$@"
