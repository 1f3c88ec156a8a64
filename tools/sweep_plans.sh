# A/B sweep of plan switches on the Swin-B / Swin-T two-kernel shapes (GPU box; output in gpurun_out/sweep.log)
o=gpurun_out/sweep.log; : > $o
for CT in "512 25088" "768 3136" "1024 6272"; do
  timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_PAIR_BN=128 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_PAIR_BN=128 SWIN_MLP_EP5_GROUPS=2 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_PAIR_BN=128 SWIN_MLP_WSL=1 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
done
