L=paper_2212_08146_b200/libkaas_b200_dev.so
for c in 2 4 5 6 3; do
 echo "== cfg $c"
 for sh in "49 512 4608" "196 256 2304" "784 128 1152"; do KAAS_LK_CFG=$c KAAS_MATMUL_LK=1 KAAS_B200_LIB=$L timeout 60 python tools/kbench.py matmul $sh 5; done
done
echo "== fc cfg 0 / 7"; for c in 0 7; do KAAS_LK_CFG=$c KAAS_MATMUL_LK=1 KAAS_B200_LIB=$L timeout 60 python tools/kbench.py matmul 1 1000 2048 5; done
