import ctypes as C, sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2604_14993_b200 import _native as N
L = N.load()
R, nd = int(sys.argv[1]), int(sys.argv[2])
keys = torch.randint(0, 2**62, (2 * R,), dtype=torch.int64, device="cuda")
out = torch.empty(R * nd + 512, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = L.cs_exp_streams(keys.data_ptr(), R, nd, out.data_ptr(), nd, 1, st.cuda_stream)
    e1.record(); torch.cuda.synchronize()
    print("plain exp_streams", R, nd, rc, round(e0.elapsed_time(e1), 3), "ms")
