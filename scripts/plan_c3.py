import sys, torch
sys.path.insert(0, ".")
from paper_2605_09755_b200.sketching import make_sketch
for (n, l) in ((2048, 500), (16384, 4000)):
    op = make_sketch("countsketch", n, l, 7, s=8)
    try:
        op.gather_plan(check=False); torch.cuda.synchronize(); print(n, l, "ok")
    except Exception as e:
        print(n, l, "ERR", e)
