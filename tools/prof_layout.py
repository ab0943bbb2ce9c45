"""One fr_layout iteration on a 100k-vertex random graph (ncu capture)."""
import sys; sys.path.insert(0, ".")
import torch
from paper_2411_09809_b200 import fr_layout
from paper_2411_09809_b200.configs import random_graph
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
fr_layout(random_graph(n, 5 * n, seed=1), iterations=1, seed=1)
torch.cuda.synchronize()
