# same-box A/B of the Jacobi in-kernel write-back (KAAS_DEV_NO_WB=1 = flush copies), bench-style
for r in 1 2 3 4; do
  for v in 0 1; do
    echo -n "no_wb=$v "; KAAS_DEV_NO_WB=$v timeout 300 python bench.py --steps 60 --warmup 5 --no-extras --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"value\", round(d[\"value\"],1), \"e2e\", round(d[\"e2e\"][\"value\"],1), \"dev p50\", round(d[\"device_p50_ms\"]*1e3,1), \"e2e p50\", round(d[\"e2e\"][\"p50_ms\"]*1e3,1), \"host\", round(d[\"e2e\"][\"host_us_per_request\"],1))"
  done
done
