#!/bin/bash
for k in mix_fwd yzt_fwd yzt_fwd_grad mix_bwd; do
  python tools/time_kernel.py $k 30
done
