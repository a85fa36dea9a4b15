import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2006_09299_b200 import Labeler, LabelingConfig
from paper_2006_09299_b200.runlab import cfg4_params
lab = Labeler(0)
idx = list(range(8)) + [97, 1023, 2048, 4095]
imgs = np.stack([O.generate(1920, 1080, *cfg4_params(i), i) for i in idx])
try:
    res = lab.label_batch(imgs, LabelingConfig())
    print("cfg4 sample ok", res.n_components[:3], "graph", lab.used_graph())
    print(lab.phase_times(0))
except Exception as e:
    traceback.print_exc()
