# same-box A/B: product vs uniform full-range fast path for the poll mask and x extraction (build/var/pfull.so)
for r in 1 2 3 4; do
  for lib in paper_2212_08146_b200/libkaas_b200.so build/var/pfull.so; do
    KAAS_B200_LIB=$lib JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500
  done
done
