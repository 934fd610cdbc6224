# dev: cGEMM A/B (per-kernel device times from an ncu launch list)
mkdir -p gpurun_out
out=gpurun_out/cgemm_ab.txt; : > $out
for lib in "" build/var/lib_cg4.so; do
  for n in 1024 2048 4096; do
    echo "== lib=${lib:-default} n=$n" >> $out
    KAAS_B200_LIB=${lib:-paper_2212_08146_b200/libkaas_b200.so} timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      python tools/kbench.py cgemm $n 5 2>/dev/null | grep -E "fused4|prep" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | sort | uniq -c | head -6 >> $out
    KAAS_B200_LIB=${lib:-paper_2212_08146_b200/libkaas_b200.so} timeout 120 python tools/kbench.py cgemm $n 5 >> $out 2>&1
  done
done
cat $out
