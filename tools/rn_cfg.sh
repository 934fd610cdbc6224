# dev: single-row tile configurations -- cfg sweep on the fc / stage-4 layers, run parity, ResNet chain
mkdir -p gpurun_out
out=gpurun_out/rn_cfg.txt; : > $out
for sub in fc s4 s3b1_3x3 s3b2_3x3; do timeout 600 python tools/run_cfg_sweep.py $sub >> $out 2>&1; done
TESTK="runs or resnet or matmul" bash tools/rn_quick.sh > /dev/null 2>&1
cat gpurun_out/rn_quick.txt >> $out
cat $out
