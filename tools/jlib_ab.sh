# same-box A/B: product vs product + cp.async shared-memory-tier fill (build/var/pcpa.so), 2 and 500 sweeps
for r in 1 2 3 4; do
  for lib in paper_2212_08146_b200/libkaas_b200.so build/var/pcpa.so; do
    for sw in 2 500; do KAAS_B200_LIB=$lib JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py $sw; done
  done
done
