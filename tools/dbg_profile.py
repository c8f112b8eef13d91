#!/usr/bin/env python
"""Debug helper: profile chosen candidates of the small YOLOX graph one at a time."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys
import paper_2406_09465_b200 as K
from korch_workloads.models import yolox_nano
ctx = K.Context(0)
kg = K.KorchGraph(ctx, yolox_nano(size=64))
cs = kg.enumerate(partition_max=64)
ids = [int(x) for x in sys.argv[1].split(",")]
for i in ids:
    print(i, kg.profile([i]), flush=True)
