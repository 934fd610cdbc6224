# same-box A/B: publishing warp 0 (product) vs 7 vs 5
for r in 1 2 3; do
  for lib in paper_2212_08146_b200/libkaas_b200.so build/var/ppub7.so build/var/ppub5.so; do
    KAAS_B200_LIB=$lib JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500
  done
done
