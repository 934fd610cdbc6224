mkdir -p gpurun_out
export KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so
{ CGAB_ONLY="pair g8,1cta g8" timeout 400 python tools/cgab.py 8192 100 6; } > gpurun_out/cgab.txt 2>&1
cat gpurun_out/cgab.txt
