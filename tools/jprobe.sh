# dev: Jacobi phase probes on the dev build (trace + compute-only timing)
mkdir -p gpurun_out
L=paper_2212_08146_b200/libkaas_b200_dev.so
{
echo "== default (product lib)"; timeout 60 python tools/kbench.py jacobi 4096 500 5
echo "== dev lib"; KAAS_B200_LIB=$L timeout 60 python tools/kbench.py jacobi 4096 500 5
echo "== dev lib, no waiting (compute + publish only; wrong results)"; KAAS_JACOBI_NOWAIT=1 KAAS_B200_LIB=$L timeout 60 python tools/kbench.py jacobi 4096 500 5
echo "== trace"; timeout 120 python tools/jtrace.py 4096; KAAS_JACOBI_TRACE=1 KAAS_JACOBI_NOWAIT=1 timeout 120 python tools/jtrace.py 4096
for v in $(ls build/var 2>/dev/null); do echo "== var $v"; KAAS_B200_LIB=build/var/$v timeout 60 python tools/kbench.py jacobi 4096 500 5; KAAS_JACOBI_NOWAIT=1 KAAS_B200_LIB=build/var/$v timeout 60 python tools/kbench.py jacobi 4096 500 5; done
} > gpurun_out/jprobe.txt 2>&1
cat gpurun_out/jprobe.txt
