"""Host enqueue time of bin_execute vs device time per step (diagnosis): if the
host needs longer to enqueue an execute than the GPU needs to run it, the
step is host-bound."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2310_02926_b200 as db
    import synth
    for wl in sys.argv[1:] or ["c2", "c3", "c5"]:
        w = synth.CONFIGS[wl]
        st = torch.cuda.Stream()
        cols = []
        for c in list(w.axes) + list(w.attrs):
            t = torch.empty(w.n, dtype=torch.float64, device="cuda")
            synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, w.n, t.data_ptr(), st.cuda_stream)
            cols.append(t)
        torch.cuda.synchronize()
        spec = db.make_spec(w.res, w.lo, w.hi, nattr=len(w.attrs), ops=w.ops)
        h = db.bin_init(spec, db.make_placement())
        hs = [db.wrap_tensor(t, stream=st.cuda_stream, mode=db.BIN_ASYNC) for t in cols]
        D = len(w.axes)
        for _ in range(5):
            t = db.bin_execute(h, hs[:D], hs[D:])
        db.bin_wait(h, t)
        K = 50
        t0 = time.perf_counter()
        for _ in range(K):
            t = db.bin_execute(h, hs[:D], hs[D:])
        t1 = time.perf_counter()
        db.bin_wait(h, t)
        t2 = time.perf_counter()
        print(f"{wl}: host enqueue {1e3 * (t1 - t0) / K:.3f} ms/execute, wall {1e3 * (t2 - t0) / K:.3f} ms/execute",
              flush=True)
        db.bin_finalize(h)
        for a in hs:
            db.bin_array_release(a)
        del cols
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
