mkdir -p gpurun_out
out=gpurun_out/jtmem.txt; : > $out
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "jacobi or Jacobi" >> $out 2>&1
for v in cols; do KAAS_JACOBI_TMEM=0 timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1 || echo "FAIL cols" >> $out; done
echo "default v6613" >> $out; timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1 || echo "FAIL v6613" >> $out
for v in v6612 v6614 v4813 v4814; do echo "$v" >> $out; KAAS_B200_LIB=build/var/lib_$v.so timeout 60 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1 || echo "FAIL $v" >> $out; done
for n in 2048 3000 4092; do timeout 60 python tools/kbench.py jacobi $n 500 3 >> $out 2>&1 || echo "FAIL n=$n" >> $out; done
cat $out
