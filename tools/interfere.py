"""Does concurrent PCIe traffic slow the tile kernels?  label_device on 8 images, alone and
while another stream copies device->host / host->device continuously."""
import sys, time, threading
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
N = 256 << 20
dbuf = torch.empty(N, dtype=torch.uint8, device="cuda"); hbuf = torch.empty(N, dtype=torch.uint8, pin_memory=True)
cs = torch.cuda.Stream()
def run(tag):
    ts = []
    for _ in range(20):
        lab.label_device(imgs.data_ptr(), S, S, 8, cfg); lab.sync(); ts.append(lab.phase_times(0).total_ms)
    ts.sort(); print(f"{tag:12s} med {ts[10]:.3f} ms  min {ts[0]:.3f}", flush=True)
run("alone")
for mode in ("d2h", "h2d"):
    with torch.cuda.stream(cs):
        for _ in range(40):
            if mode == "d2h": hbuf.copy_(dbuf, non_blocking=True)
            else: dbuf.copy_(hbuf, non_blocking=True)
    run(mode)
    torch.cuda.synchronize()
run("alone")
