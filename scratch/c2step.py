import sys, time, torch
sys.path.insert(0, '.')
import paper_2210_15114_b200 as l1
from paper_2210_15114_b200 import workloads as wl
from paper_2210_15114_b200.distributed import ShardedL1DM
w = wl.workload("c2")
X = wl.make_points(w, "cuda"); Zs = [wl.make_query(w, t, "cuda") for t in range(20)]
Y = torch.empty((w.n, 1), dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    sh = ShardedL1DM(X, k_range=(0, 64), stream=stream)
    e[1].record(); t1 = time.perf_counter()
    l1.l1dm_timing_enable(sh.handle, True)
    for q in range(20): sh.matvec(Zs[q], Y, root=0, overlap_blocks=4)
    e[2].record(); t2 = time.perf_counter()
    tr = l1.l1dm_timing_read(sh.handle); t3 = time.perf_counter()
    sh.close(); e[3].record(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"gpu: prep {e[0].elapsed_time(e[1]):.2f} queries {e[1].elapsed_time(e[2]):.2f} close {e[2].elapsed_time(e[3]):.2f} | host: prep {1e3*(t1-t0):.2f} enqueue {1e3*(t2-t1):.2f} tread {1e3*(t3-t2):.2f} close {1e3*(t4-t3):.2f} | lib prep {tr['prep_ms']:.2f}")
