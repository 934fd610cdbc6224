# cGEMM 1024^3: split-K 2 (default) vs narrow N128 tiles vs CTA pair, GEMM kernel time under ncu (dev build)
export KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so
for v in "def:" "narrow:KAAS_CGEMM_KSPLIT=0" "pair:KAAS_CGEMM_PAIR=1"; do
  name=${v%%:*}; envs=${v#*:}
  echo "== $name"
  env $envs timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/kbench.py cgemm 1024 3 2>/dev/null | grep -i "k_cgemm\|memset" | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | sort | uniq -c | head -8
  env $envs timeout 120 python tools/kbench.py cgemm 1024 20
done
