import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import hytgen, paper_2208_14935_b200 as hyt
from bench import pin_host
g = hytgen.make("tw", weighted=True)
pin_host([g.off, g.nbr, g.w])
for weighted in (False, True, False, True):
    G = hyt.Graph(device=0, budget=16 << 30)
    t = time.time()
    G.load(g.off, g.nbr, g.w if weighted else None)
    print("weighted" if weighted else "ids only", "load_s", round(time.time() - t, 3), flush=True)
    G.close()
