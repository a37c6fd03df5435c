#!/bin/bash
# Depth-chunk boundary sweep (SGS_DEPTH_CHUNKS) at config C.
for c in "16,4" "16" "8" "32,4" "16,4,2" "32,8,2" "64,16,4" "24,6"; do
  echo "chunks $c"; SGS_DEPTH_CHUNKS=$c python tools/quick_time.py 2>&1 | grep -E "V P|preprocess|batch32 device"
done
