# dev: Jacobi parity subset + kernel-only timing (A/B against build/var libs)
mkdir -p gpurun_out
out=gpurun_out/jvar.txt; : > $out
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "jacobi or Jacobi" 2>&1 | tail -2 >> $out
for i in 1 2 3; do echo "== default" >> $out; timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1; done
for v in $(ls build/var 2>/dev/null); do echo "== $v" >> $out; KAAS_B200_LIB=build/var/$v timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1 || echo FAIL >> $out; done
cat $out
