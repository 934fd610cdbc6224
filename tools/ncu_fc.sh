mkdir -p gpurun_out
for shp in "1 1000 2048" "49 512 4608"; do
  tag=$(echo $shp | tr ' ' x)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_run" -s 4 -c 1 -f \
    -o gpurun_out/run_$tag python tools/mm_one.py $shp 6 > gpurun_out/ncu_run_$tag.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
