for i in 1 2; do
python tools/probe.py c2 | cut -c1-40
GT_NO_EARLY_OAA=1 python tools/probe.py c2 | cut -c1-60
GT_OAA_MAXLEVEL=5 python tools/probe.py c2 | cut -c1-60
GT_OAA_MAXLEVEL=4 python tools/probe.py c2 | cut -c1-60
GT_OAA_CTAS=148 python tools/probe.py c2 | cut -c1-60
GT_OAA_CTAS=296 python tools/probe.py c2 | cut -c1-60
GT_OAA_CTAS=592 python tools/probe.py c2 | cut -c1-60
GT_OAA_CTAS=1184 python tools/probe.py c2 | cut -c1-60
done
