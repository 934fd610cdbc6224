# cGEMM CTA-pair A/B: correctness, kernel times pair vs 1-CTA, DRAM bytes of one pair launch
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "cgemm" 2>&1 | tail -4
for n in 2048 4096 8192; do
  echo "== n=$n pair"; timeout 120 python tools/kbench.py cgemm $n 10
  echo "== n=$n 1-CTA (dev)"; KAAS_CGEMM_PAIR=0 KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so timeout 120 python tools/kbench.py cgemm $n 10
done
timeout 300 ncu --set full --clock-control none -k regex:k_cgemm_pair -c 1 -o gpurun_out/cgpair8192 -f python tools/kbench.py cgemm 8192 1 > gpurun_out/ncu_cgpair.log 2>&1; echo "ncu rc=$?"
} > gpurun_out/cgpair.txt 2>&1
cat gpurun_out/cgpair.txt
