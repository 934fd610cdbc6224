# same-box A/B: product vs branch-free pending update + trap check every 256 polls (build/var/ppoll.so)
for r in 1 2 3 4; do
  for lib in paper_2212_08146_b200/libkaas_b200.so build/var/ppoll.so; do
    KAAS_B200_LIB=$lib JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500
  done
done
