import time, numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2210_08804_b200 as hps, bench
v = hps.VolatileStore(8)
t = hps.TableId("x", 128)
v.register_table(t, hps.VolatileTableConfig(partition_count=16, overflow_margin=1<<40))
keys = np.arange(2_000_000, dtype=np.uint64) * np.uint64(2654435761)
for i in range(0, len(keys), 1<<18):
    k = keys[i:i+(1<<18)]; v.insert("x", k, bench.table_rows(k, 128))
rng = np.random.default_rng(0)
q = keys[rng.integers(0, len(keys), 65536)]
v.lookup("x", q)
t0 = time.perf_counter()
for _ in range(10): r = v.lookup("x", q)
print("lookup 65536 x d128: %.2f ms" % ((time.perf_counter()-t0)*100))
import ctypes as C, torch
# pinned destination, like the refresh / engine staging
d = 128
fk = torch.empty(65536, dtype=torch.int64).pin_memory()
fv = torch.empty(65536 * d).pin_memory()
mk = torch.empty(65536, dtype=torch.int64).pin_memory()
nf, nm = C.c_size_t(0), C.c_size_t(0)
qq = np.ascontiguousarray(q)
for rep in range(2):
    t0 = time.perf_counter()
    for _ in range(10):
        hps.lib().hps_vdb_lookup(v.handle, b"x", qq.ctypes.data, len(qq), fk.data_ptr(), fv.data_ptr(), C.byref(nf), mk.data_ptr(), C.byref(nm))
    print("pinned-destination lookup: %.2f ms (found %d)" % ((time.perf_counter()-t0)*100, nf.value))
