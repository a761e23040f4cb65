"""DMMA GEMM with C in local HBM vs C in the peer GPU's HBM (the inbox path).

One process, two GPUs, no NCCL: td_peer_enable + td_peer_alloc on GPU 1,
td_dgemm on GPU 0 writing its epilogue tiles over NVLink.  If the two times
agree, the reduce write-back of a Johnson / COSMA partial costs nothing on
top of the GEMM that produces it.
"""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2203_08069_b200 import _native as nat  # noqa: E402

nat.load()
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def gen(shape, tid, dev):
    t = torch.empty(shape, dtype=torch.float64, device=dev)
    st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    nat.call("td_generate", st, len(shape), nat.i64_array(shape), nat.i64_array([0] * len(shape)),
             nat.i64_array(shape), P(t), nat.i64_array(t.stride()), 0, tid, 0)
    return t


def main():
    M = N = 16384
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    torch.cuda.set_device(0)
    a, b = gen((M, K), 1, d0), gen((K, N), 2, d0)
    c_local = torch.empty((M, N), dtype=torch.float64, device=d0)
    nat.call("td_peer_enable", 0, 1)
    ptr = C.c_void_p()
    nat.call("td_peer_alloc", 1, M * N * 8, C.byref(ptr), None)
    st = C.c_void_p(torch.cuda.current_stream(d0).cuda_stream)

    def run(cptr):
        nat.call("td_dgemm", st, M, N, K, P(a), K, P(b), N, cptr, N, 0)

    res = {}
    for name, cptr in (("local", P(c_local)), ("peer", ptr), ("local2", P(c_local)), ("peer2", ptr)):
        run(cptr)
        torch.cuda.synchronize(d0)
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run(cptr)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ms = sorted(ts)[len(ts) // 2]
        res[name] = {"ms": ms, "tflops": 2.0 * M * N * K / ms / 1e9}
        print(name, res[name], flush=True)
    # the peer copy holds the same product
    peer_view = torch.empty((M, N), dtype=torch.float64, device=d1)
    nat.call("td_memcpy_2d", C.c_void_p(torch.cuda.current_stream(d1).cuda_stream), P(peer_view), N, ptr, N, N, M)
    torch.cuda.synchronize(d1)
    res["same_bits"] = bool(torch.equal(peer_view.to(d0), c_local))
    res["bytes_to_peer_per_launch"] = M * N * 8
    print(json.dumps(res))
    json.dump(res, open("gpurun_out/peer_gemm.json", "w"), indent=1)
    nat.call("td_peer_free", 1, ptr)


if __name__ == "__main__":
    main()
