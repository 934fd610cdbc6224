for x in 0 1; do for st in 8 12; do
  echo "XREG=$x STAGES=$st"; KAAS_JACOBI_XREG=$x KAAS_JACOBI_STAGES=$st python tools/kbench.py jacobi 4096 500 3
done; done > gpurun_out/jab.log 2>&1
KAAS_JACOBI_XREG=0 KAAS_JACOBI_STAGES=8 ncu --set full --import-source on --clock-control none -k regex:jacobi_tma -c 1 -o gpurun_out/jac_x0s8 python tools/kbench.py jacobi 4096 100 1 > /dev/null 2>&1
KAAS_JACOBI_XREG=1 KAAS_JACOBI_STAGES=12 ncu --set full --import-source on --clock-control none -k regex:jacobi_tma -c 1 -o gpurun_out/jac_x1s12 python tools/kbench.py jacobi 4096 100 1 > /dev/null 2>&1
