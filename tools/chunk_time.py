import torch, sys
sys.path.insert(0, "/root/repo")
from paper_2006_09299_b200 import Labeler, LabelingConfig
from paper_2006_09299_b200.runlab import cfg2_cells, generate_device
cells = list(cfg2_cells()); B = len(cells); S = 2048
imgs = torch.empty((B, S, S), dtype=torch.uint8, device="cuda")
for i, (d, g) in enumerate(cells): generate_device(imgs[i].data_ptr(), S, S, d, g, 1)
cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
lab = Labeler(0)
for n in (8, 16, 35, 105):
    for b0 in (0, 48):
        if b0 + n > B: continue
        ts = []
        for _ in range(6):
            lab.label_device(imgs[b0].data_ptr(), S, S, n, cfg); lab.sync(); ts.append(lab.phase_times(0).total_ms)
        t = sorted(ts)[2]
        print(f"n={n:3d} b0={b0:3d}: {t:.3f} ms  {n*S*S/t/1e6:.1f} Gpx/s  graph={lab.used_graph()}")
