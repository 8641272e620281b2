import sys; sys.path.insert(0, '.')
import torch
from paper_2302_01838_b200 import LossWeights, ModelArch, init_stacked, train_on_batch
from paper_2302_01838_b200.trainer import _synthetic_batch
arch = ModelArch(n_layers=4, hidden=128, n_freq=5)
params, state = init_stacked(arch, 1, seed=11)
batch = _synthetic_batch(arch, 1, int(sys.argv[1]) if len(sys.argv) > 1 else 300, 10, seed=7)
print(train_on_batch(params, state, batch, LossWeights()))
torch.cuda.synchronize(); print("ok")
