# A/B sweep of plan switches on the Swin-B / Swin-T two-kernel shapes (GPU box; output in gpurun_out/sweep.log)
o=gpurun_out/sweep.log; : > $o
for CT in "384 12544" "512 12544" "512 25088" "384 50176" "448 12544"; do
  timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_LN_PAIR=0 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
done
