"""Plan build + pack vs loading the device-ready program cache (BFLYSHT1)."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0910_5435_b200 as bb
l = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
t = time.time(); sht = bb.SHT(l, eps=1e-12); t_build = time.time() - t
path = os.path.join(tempfile.gettempdir(), f"sht{l}.bflysht")
t = time.time(); sht.save(path); t_save = time.time() - t
del sht
t = time.time(); again = bb.SHT.load(path); torch.cuda.synchronize(); t_load = time.time() - t
print(f"l={l}: build+pack+upload {t_build:.1f} s, save {t_save:.1f} s ({os.path.getsize(path) / 1e9:.2f} GB), load {t_load:.1f} s")
os.remove(path)
