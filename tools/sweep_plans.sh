# A/B: relaxed vs release remote arrive of the pair's TMEM-drained signal (GPU box; gpurun_out/sweep.log)
o=gpurun_out/sweep.log; : > $o
for CT in "512 25088" "768 3136" "1024 6272" "512 12544"; do
  timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
  SWIN_MLP_DBG1=16 timeout 120 python tools/layer_sweep.py $CT >> $o 2>&1
done
