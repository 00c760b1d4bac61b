import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from conftest import c1_images
import paper_1711_01919_b200 as ih
from paper_1711_01919_b200 import device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for idx, (w, h, b, tile, px) in enumerate(c1_images(200)):
    if idx >= n: break
    img, spec = ih.GrayImage(px), ih.BinSpec.uniform(b)
    for name, fn in [("seq", lambda: ih.compute_sequential(img, spec)), ("cw", lambda: ih.compute_crossweave(img, spec))]:
        print(idx, w, h, b, name, flush=True)
        r = fn(); torch.cuda.synchronize(); r.counts
