# dev: Jacobi A/B of build/var libs against the default (same box, alternating), parity first
mkdir -p gpurun_out
out=gpurun_out/jvar.txt; : > $out
for v in $(ls build/var 2>/dev/null); do
  echo "== parity $v" >> $out
  KAAS_B200_LIB=build/var/$v timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "jacobi_config2 or jacobi_edge or every_residual or onchip" 2>&1 | tail -1 >> $out
done
for i in 1 2; do
  echo "== default" >> $out; timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1
  for v in $(ls build/var 2>/dev/null); do echo "== $v" >> $out; KAAS_B200_LIB=build/var/$v timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1 || echo FAIL >> $out; done
done
cat $out
