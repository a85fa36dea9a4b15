"""D2H bandwidth alone and while the tile kernels run on another stream."""
import sys, threading, time
import torch
sys.path.insert(0, "/root/repo")
from paper_2006_09299_b200 import Labeler, LabelingConfig
from paper_2006_09299_b200.runlab import cfg2_cells, generate_device
cells = list(cfg2_cells()); S = 2048
imgs = torch.empty((8, S, S), dtype=torch.uint8, device="cuda")
for i in range(8):
    d, g = cells[48 + i]; generate_device(imgs[i].data_ptr(), S, S, d, g, 1)
cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
lab = Labeler(0)
N = 24 << 20
dbuf = torch.empty(N, dtype=torch.uint8, device="cuda"); hbuf = torch.empty(N, dtype=torch.uint8, pin_memory=True)
cs = torch.cuda.Stream()
def d2h(tag, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    with torch.cuda.stream(cs):
        for _ in range(reps): hbuf.copy_(dbuf, non_blocking=True)
    e1.record(cs)
    return e0, e1, reps
e0, e1, r = d2h("alone"); torch.cuda.synchronize(); print(f"alone: {r*N/e0.elapsed_time(e1)/1e6:.1f} GB/s")
e0, e1, r = d2h("busy")
for _ in range(30):
    lab.label_device(imgs.data_ptr(), S, S, 8, cfg)
torch.cuda.synchronize(); print(f"with kernels: {r*N/e0.elapsed_time(e1)/1e6:.1f} GB/s")
