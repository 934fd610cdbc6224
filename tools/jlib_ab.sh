# same-box A/B: product library vs the previous commit's product build (build/var/pold.so)
for r in 1 2 3 4; do
  for lib in build/var/pold.so paper_2212_08146_b200/libkaas_b200.so; do
    KAAS_B200_LIB=$lib JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500
  done
done
