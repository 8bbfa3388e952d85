# power iteration through DistributedArgCsr with the engine converted on a side stream (the bench's setup)
import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_1203_5737_b200.multigpu import DistributedArgCsr
from paper_1203_5737_b200 import synthetic
dev = torch.device("cuda", 0)
for n in (30, 100):
    A = synthetic.stencil3d27(n, dev)
    x0 = synthetic.bench_input(A.num_cols, dev, torch.float64)
    out = []
    for ex in ["auto", "p2p"]:
        side = torch.cuda.Stream(dev)
        with torch.cuda.stream(side):
            D = DistributedArgCsr(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, 128, 1, device=dev, exchange=ex)
        out.append(D.power_iteration(x0.clone(), 33)[0])
        D.close()
    print(n, out)
