# DRAM bytes + time per cGEMM 8192 launch vs raster group size, pair vs 1-CTA (dev lib)
mkdir -p gpurun_out
export KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so
{
for pair in 1 0; do for g in 1 2 4 8 16 32; do
  echo "== pair=$pair group=$g"
  KAAS_CGEMM_PAIR=$pair KAAS_CGEMM_GROUPM=$g timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_cgemm -c 2 python tools/kbench.py cgemm 8192 1 2>&1 | grep -E "dram__|gpu__time|hit_rate"
  KAAS_CGEMM_PAIR=$pair KAAS_CGEMM_GROUPM=$g timeout 120 python tools/kbench.py cgemm 8192 10
done; done
} > gpurun_out/cggroup2.txt 2>&1
cat gpurun_out/cggroup2.txt
