# A/B of TMEM-kernel variants (dev build, KAAS_JACOBI_TMV=RR,MODE,DEP), interleaved, L2-flushed chains
for r in 1 2 3; do
  for v in 6,1,4 def 6,3,4 6,3,6 5,3,5 5,3,6 7,3,5; do
    echo -n "TMV=$v  "; if [ $v = def ]; then JPRO_REPS=21 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500; else KAAS_JACOBI_TMV=$v JPRO_REPS=21 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500; fi
  done
done
