set -x
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "jacobi" 2>&1 | tail -2
for i in 1 2; do
  for v in paper_2212_08146_b200/libkaas_b200.so build/var/oldfill.so; do
    echo "== $v"; KAAS_B200_LIB=$v timeout 300 python tools/jhost.py
  done
done
