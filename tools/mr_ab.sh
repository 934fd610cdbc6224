# same-box A/B of k_jacobi_tmem register caps (tools/build_pvar.sh variants), full warm request path
for r in 1 2 3; do
  for v in base mr248 mr240 mr232; do
    echo -n "$v round $r: "; KAAS_B200_LIB=build/var/$v.so timeout 200 python tools/spec_ab.py --off-only 2>&1 | grep "speculative="
  done
done
