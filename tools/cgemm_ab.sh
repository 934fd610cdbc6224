# dev: cGEMM A/B (per-kernel device times from an ncu launch list + kbench wall)
mkdir -p gpurun_out
out=gpurun_out/cgemm_ab.txt; : > $out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "cgemm" 2>&1 | tail -2 >> $out
for ks in 1 0; do
  for n in 512 1024 1536; do
    echo "== KSPLIT=$ks n=$n" >> $out
    KAAS_CGEMM_KSPLIT=$ks timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      python tools/kbench.py cgemm $n 5 2>/dev/null > gpurun_out/ncu_tmp.csv
    python - >> $out <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/ncu_tmp.csv")) if len(r) > 14 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4].split("(")[0]].append(float(r[14]) / 1e3)
for k, v in agg.items():
    v.sort()
    print(f"   {k:60s} n={len(v)} median {v[len(v)//2]:8.1f} us")
PY
    KAAS_CGEMM_KSPLIT=$ks timeout 120 python tools/kbench.py cgemm $n 10 >> $out 2>&1
  done
done
cat $out
