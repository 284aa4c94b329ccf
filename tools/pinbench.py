import time, numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_1803_09835_b200 import lsh_search as ls
n = 8_640_000
d = torch.randint(0, 4096, (86391, 200), dtype=torch.int32, device="cuda")
x = np.random.default_rng(0).standard_normal(n)
for it in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); b = torch.empty(d.shape, dtype=d.dtype, pin_memory=True); t1=time.perf_counter(); b.copy_(d); t2=time.perf_counter()
    print("pin alloc %.2f ms, d2h %.2f ms" % ((t1-t)*1e3, (t2-t1)*1e3))
    pool = ls._copy_pool()
    t=time.perf_counter(); out = np.empty(d.shape, np.int32); hb = b.numpy(); step = -(-d.shape[0]//8)
    list(pool.map(lambda i: np.copyto(out[i:i+step], hb[i:i+step]), range(0, d.shape[0], step))); t1=time.perf_counter()
    print("np.empty+threaded copy %.2f ms" % ((t1-t)*1e3))
    t=time.perf_counter(); xd = ls._to_device_staged(x); torch.cuda.synchronize(); t1=time.perf_counter()
    print("staged h2d 69MB %.2f ms" % ((t1-t)*1e3))
    t=time.perf_counter(); xp = torch.from_numpy(x).pin_memory(); t1=time.perf_counter()
    print("pin 69MB copy %.2f ms" % ((t1-t)*1e3))
