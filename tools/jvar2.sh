# dev: A/B the TMEM-tier Jacobi variants (KAAS_JACOBI_TMV="RR,MODE,DEP", dev build)
mkdir -p gpurun_out
L=paper_2212_08146_b200/libkaas_b200_dev.so
VARS=${VARS:-"6,0,4 6,1,2 6,1,3 6,1,4 7,1,2 8,1,2 8,1,3 9,1,2"}
out=gpurun_out/jvar2.txt; : > $out
for v in $VARS; do
  echo "== parity $v" >> $out
  KAAS_JACOBI_TMV=$v KAAS_B200_LIB=$L timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "jacobi_config2 or jacobi_edge or every_residual or onchip or repeated" 2>&1 | tail -1 >> $out
done
for rep in 1 2; do
  for v in $VARS; do
    echo "== $v" >> $out; KAAS_JACOBI_TMV=$v KAAS_B200_LIB=$L timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1
  done
done
for v in $VARS; do
  echo "== trace $v" >> $out; KAAS_JACOBI_TMV=$v timeout 60 python tools/jtrace.py 4096 2>&1 | grep -v "^jacobi" >> $out
done
cat $out
