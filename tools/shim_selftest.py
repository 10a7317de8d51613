"""Two-process self test of tests/nccl_shim (GPU): grouped send/recv and all-reduce."""
import ctypes as C, multiprocessing as mp, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "nccl_shim", "libnccl_shim.so")

def rank(r, uid, q):
    import torch
    torch.cuda.set_device(0)
    L = C.CDLL(SHIM)
    comm = C.c_void_p()
    idb = (C.c_char * 128).from_buffer_copy(uid)
    class Uid(C.Structure): _fields_ = [("internal", C.c_char * 128)]
    u = Uid(); C.memmove(C.addressof(u), uid, 128)
    L.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, Uid, C.c_int]
    rc = L.ncclCommInitRank(C.byref(comm), 2, u, r)
    s = torch.cuda.Stream()
    a = torch.arange(10, dtype=torch.float32, device="cuda") + 100 * r
    b = torch.full((10,), -1.0, dtype=torch.float32, device="cuda")
    d = torch.tensor([1.5 + r, 2.0 * r], dtype=torch.float64, device="cuda")
    m = torch.tensor([7 + r], dtype=torch.int32, device="cuda").view(torch.int32)
    L.ncclSend.argtypes = L.ncclRecv.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    L.ncclAllReduce.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    torch.cuda.synchronize()
    rcs = [rc]
    rcs.append(L.ncclGroupStart())
    rcs.append(L.ncclSend(a.data_ptr(), 10, 7, 1 - r, comm, s.cuda_stream))
    rcs.append(L.ncclRecv(b.data_ptr(), 10, 7, 1 - r, comm, s.cuda_stream))
    rcs.append(L.ncclGroupEnd())
    rcs.append(L.ncclAllReduce(d.data_ptr(), d.data_ptr(), 2, 8, 0, comm, s.cuda_stream))
    rcs.append(L.ncclAllReduce(m.data_ptr(), m.data_ptr(), 1, 3, 2, comm, s.cuda_stream))
    torch.cuda.synchronize()
    q.put((r, rcs, b.cpu().tolist(), d.cpu().tolist(), m.cpu().tolist()))
    L.ncclCommDestroy(comm)

if __name__ == "__main__":
    L = C.CDLL(SHIM); buf = C.create_string_buffer(128); L.ncclGetUniqueId(buf)
    c = mp.get_context("spawn"); q = c.Queue()
    ps = [c.Process(target=rank, args=(r, buf.raw[:128], q)) for r in range(2)]
    [p.start() for p in ps]
    for _ in range(2): print(q.get(timeout=60))
    [p.join() for p in ps]
