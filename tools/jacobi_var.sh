# dev: ncu capture of the Jacobi TMEM kernel
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"jacobi_tmem" -c 1 \
    -o gpurun_out/jtmem_full -f python tools/kbench.py jacobi 4096 500 1 > gpurun_out/ncu_jtmem.log 2>&1
tail -5 gpurun_out/ncu_jtmem.log
