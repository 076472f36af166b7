import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_0910_5435_b200 as bb
from oracle import sht_oracle
l, B = int(sys.argv[1]), int(sys.argv[2])
os.environ["BFLY_WAVES"] = "1"
s = bb.SHT(l, eps=1e-12)
beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=1)).cuda()
g = s.synthesize(beta); torch.cuda.synchronize(); print("synth ok", flush=True)
b = s.analyze(g); torch.cuda.synchronize(); print("anal ok", float((torch.linalg.vector_norm(b-beta)/torch.linalg.vector_norm(beta)).item()), flush=True)
