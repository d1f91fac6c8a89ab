for mb in 32 64 128 256; do
  echo "== GT_LA8_MB=$mb"
  GT_LA8_MB=$mb timeout 300 python tools/c4_breakdown.py
  GT_LA8_MB=$mb QT_TRAIN_ONLY=1 timeout 200 python tools/quick_time.py | grep -E "per-kernel|train ms"
done
