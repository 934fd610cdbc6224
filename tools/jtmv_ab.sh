# A/B of TMEM-kernel variants (dev build, KAAS_JACOBI_TMV=RR,MODE,DEP), interleaved, L2-flushed chains
for r in 1 2 3; do
  for v in def 6,4,5 6,4,4 5,4,5; do
    echo -n "TMV=$v  "; if [ $v = def ]; then JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500; else KAAS_JACOBI_TMV=$v JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500; fi
  done
done
for v in 6,4,5 5,4,5; do
  KAAS_JACOBI_TMV=$v timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "jacobi" 2>&1 | tail -1
done
