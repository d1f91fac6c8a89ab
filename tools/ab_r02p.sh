python tools/probe.py c2
GT_PART_NO_BALANCE=1 python tools/probe.py c2
GT_FUSED_NO_XPRE=1 python tools/probe.py c2
GT_PART_NO_BALANCE=1 GT_FUSED_NO_XPRE=1 python tools/probe.py c2
python tools/probe.py c2
python tools/probe.py walk
GT_WALK_TPB=128 python tools/probe.py walk
python tools/probe.py c4
