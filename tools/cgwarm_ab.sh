export KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so
for r in 1 2 3 4; do
for gp in "8 8" "4 2" "8 2"; do
  set -- $gp
  KAAS_CGEMM_GROUPM=$1 KAAS_CGEMM_PANELM=$2 timeout 300 python tools/cgwarm_ab.py 2>/dev/null | tail -1
done
done
