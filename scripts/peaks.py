import sys; sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D
import torch
torch.cuda.init()
for it in (100000, 400000):
    print("dmma", it, [round(D.peak_dmma_tflops(0, it), 2) for _ in range(3)])
    print("dfma", it, [round(D.peak_dfma_tflops(0, it), 2) for _ in range(3)])
