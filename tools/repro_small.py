import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_22265_b200 as ebcc
from paper_2510_22265_b200 import fields
for (r, c) in [(8, 8), (16, 16), (24, 24), (33, 17)]:
    a = fields.small_field("smooth", r, c, 1)
    print(r, c, len(ebcc.compress(a, 0.01)), flush=True)
