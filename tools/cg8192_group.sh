# cGEMM 8192^3 raster group size (dev knob KAAS_CGEMM_GROUPM): DRAM bytes + time under ncu, and kbench timing
export KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so
for g in 8 4 12 16 24; do
  echo "== group $g"
  KAAS_CGEMM_GROUPM=$g timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_cgemm_fused4 -c 1 python tools/kbench.py cgemm 8192 1 2>/dev/null | grep -E "dram__bytes_read|gpu__time_duration|cycles_elapsed"
  KAAS_CGEMM_GROUPM=$g timeout 200 python tools/kbench.py cgemm 8192 8
done
