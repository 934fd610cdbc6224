L=paper_2212_08146_b200/libkaas_b200_dev.so
for g in 8 16 32 64 4; do echo "== group $g"; KAAS_CGEMM_GROUPM=$g KAAS_B200_LIB=$L timeout 120 python tools/kbench.py cgemm 8192 5; done
for g in 8 32; do KAAS_CGEMM_GROUPM=$g KAAS_B200_LIB=$L timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second -k regex:k_cgemm_fused4 -s 1 -c 1 python tools/kbench.py cgemm 8192 1 2>&1 | grep -E "dram__bytes|duration|per_second"; done
