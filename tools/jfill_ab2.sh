# A/B: Jacobi chain (500 sweeps, L2 flushed) old vs new build, interleaved
for r in 1 2 3; do
  for lib in build/var/jhead.so paper_2212_08146_b200/libkaas_b200_dev.so; do
    for sw in 2 500; do KAAS_B200_LIB=$lib JPRO_REPS=21 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py $sw; done
  done
done
