import sys
sys.path.insert(0,'tests'); sys.path.insert(0,'oracle'); sys.path.insert(0,'.')
import numpy as np, golden_io, torch
import paper_2406_11209_b200 as bz
from test_gpu_golden import ref_compressed
ops=[c for c in golden_io.op_cases() if c["name"]=="ops_c5"][0]
a=ref_compressed(bz, golden_io.compress_case(ops["a"])); b=ref_compressed(bz, golden_io.compress_case(ops["b"]))
ref=ops["arrays"]
for name, c in (("sub", bz.subtract(a,b)), ("addneg", bz.add(a, bz.negate(b))), ("add", bz.add(a,b))):
    tag = "add" if name=="add" else "sub"
    gm=c.maxima_f64().cpu().numpy().reshape(-1); wm=ref[f"{tag}_max"].reshape(-1)
    gi=c.indices.cpu().numpy().reshape(gm.size,-1); wi=ref[f"{tag}_idx"].reshape(gm.size,-1)
    badm=np.nonzero(gm!=wm)[0]; badi=np.nonzero((gi!=wi).any(1))[0]
    print(name, "bad maxima blocks", badm, "bad idx blocks", badi)
    for blk in badm[:3]:
        print("  blk", blk, gm[blk], wm[blk])
