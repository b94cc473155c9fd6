import ctypes, os, sys
import numpy as np, torch
os.environ["ESM_ATTN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10548_b200 import _lib
from paper_2411_10548_b200.model import rope_tables
lib = _lib.load()
B, nh, S, dh = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,20,1024,24").split(",")]
H = nh * dh
st = torch.cuda.current_stream().cuda_stream
q, k, v = ((torch.randn(B, nh, S, dh, device="cuda") * 0.5).bfloat16() for _ in range(3))
am = torch.ones(B, S, dtype=torch.int32, device="cuda")
o = torch.empty(B * S, H, device="cuda", dtype=torch.bfloat16); lse = torch.empty(B, nh, S, device="cuda")
_lib.call("esm_attn_fwd", 1, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), o.data_ptr(), lse.data_ptr(), B, nh, S, dh, st)
do = torch.randn(B * S, H, device="cuda").bfloat16()
cos, sin = (torch.from_numpy(t).cuda() for t in rope_tables(S, dh))
delta = torch.empty(2, B, nh, S, device="cuda"); ws = torch.empty(B * S, H, device="cuda")
dqkv = torch.empty(B * S, 3 * H, device="cuda", dtype=torch.bfloat16); cs = torch.zeros(3 * H, device="cuda")
for _ in range(3):
    _lib.call("esm_attn_bwd_qkv", q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), am.data_ptr(), delta.data_ptr(), ws.data_ptr(), dqkv.data_ptr(), cs.data_ptr(), cos.data_ptr(), sin.data_ptr(), dh ** -0.5, B, nh, S, dh, st)
torch.cuda.synchronize()
buf = np.zeros(3 * 64 * 8, dtype=np.uint64)
lib.esm_debug_attn_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.esm_debug_attn_trace(buf.ctypes.data))
t = buf.reshape(3, 64, 8).astype(np.int64)
t0 = t[t > 0].min()
names = {0: ["wait_ds", "ds_ok", "dvdk_issued", "s_next_issued"], 1: ["wait_s", "s_ok", "ld_done", "comp_done", "bar_done", "arrived", "drained"]}
names[2] = names[1]
nb = S // 64
for r in range(3):
    print("role", r)
    for i in range(min(nb, 16)):
        ev = t[r, i]
        n = names[r]
        print(f"  blk {i:2d} " + " ".join(f"{n[e]}={(ev[e]-t0) if ev[e] else -1:7d}" for e in range(len(n))))
