python -m pytest tests/test_gpu.py -q -x -k "inference" 2>&1 | tail -2
GT_WALK_SPLIT=8 python -m pytest tests/test_gpu.py -q -x -k "inference" 2>&1 | tail -2
GT_WALK_SPLIT=2 python -m pytest tests/test_gpu.py -q -x -k "inference" 2>&1 | tail -2
python tools/probe.py walk
for v in 1 2 4 8 16; do GT_WALK_SPLIT=$v python tools/probe.py walk; done
