# A/B sweep of plan switches for the one-window config (T = 49) (GPU box; output in gpurun_out/sweep.log)
o=gpurun_out/sweep.log; : > $o
for CT in "768 49" "768 3136"; do
  timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_LN_CS=8 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_PAIR=0 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_PAIR=0 SWIN_MLP_LN_CS=8 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_PAIR=0 SWIN_MLP_LN_CS=8 SWIN_MLP_NO_RESB=1 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
done
