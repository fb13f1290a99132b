# fwd MMA issuer: one continuous tile stream across work items (the next item's S tiles are
# issued LAG ahead of the PV side instead of after the current item's last PV)
import os
HERE = os.path.dirname(os.path.abspath(__file__))
OLD = open(os.path.join(HERE, "fwd_xitem_old.cu.txt")).read()
NEW = open(os.path.join(HERE, "fwd_xitem.cu.txt")).read()
PATCHES = [("attn_fwd_sm100.cu", OLD, NEW)]
