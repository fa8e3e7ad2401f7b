"""e2e study (r02b): pinned-host copy bandwidths on this box (H2D alone, D2H
alone, both at once) for the batched layer's In / Out sizes, and
conv_run_host's step time for a path at several chunk counts
(CONV_HOST_CHUNKS is read once per process, so each count runs in its own
subprocess).  Usage: python scripts/probe_e2e.py [path] [config]"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def copies(bi, bo, n=10):
    dev = torch.device("cuda", 0)
    hi = torch.empty(bi // 4, dtype=torch.float32).pin_memory()
    ho = torch.empty(bo // 4, dtype=torch.float32).pin_memory()
    di = torch.empty(bi // 4, dtype=torch.float32, device=dev)
    do = torch.empty(bo // 4, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, ops in (("h2d", [(s1, di, hi)]), ("d2h", [(s2, ho, do)]), ("both", [(s1, di, hi), (s2, ho, do)])):
        for _ in range(2):
            for s, dst, src in ops:
                with torch.cuda.stream(s):
                    dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        for _ in range(n):
            for s, dst, src in ops:
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    dst.copy_(src, non_blocking=True)
            for s, _, _ in ops:
                cur.wait_stream(s)
        b.record(cur)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        nbytes = sum(dst.numel() * 4 for _, dst, _ in ops)
        res[name] = {"ms": round(ms, 4), "GB/s": round(nbytes / ms / 1e6, 1)}
    return res


def one(path, cfg, chunks):
    from paper_2101_09808_b200 import conv
    from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
    sh = CONFIGS[cfg]
    xi, wi = make_inputs(sh, seed=0)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path)
    xi, wi = xi.pin_memory(), wi.pin_memory()
    out = torch.empty(sh.out_shape, dtype=torch.float32).pin_memory()
    dbuf = torch.empty(plan.host_run_bytes, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        plan.run_host(xi, wi, out, dbuf)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    a.record()
    for _ in range(n):
        plan.run_host(xi, wi, out, dbuf)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    return {"path": path, "chunks": chunks, "ms": round(ms, 4), "tflops": round(sh.flops / ms / 1e9, 2)}


if __name__ == "__main__" and not os.environ.get("PROBE_COPY_PIPELINE") and not os.environ.get("PROBE_COPY_LOAD") and not os.environ.get("PROBE_OVERLAP"):
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        print(json.dumps(one(sys.argv[2], sys.argv[3], os.environ.get("CONV_HOST_CHUNKS", "auto"))), flush=True)
        sys.exit(0)
    path = sys.argv[1] if len(sys.argv) > 1 else "fp32_simt"
    cfg = sys.argv[2] if len(sys.argv) > 2 else "batched"
    from paper_2101_09808_b200.inputs import CONFIGS
    sh = CONFIGS[cfg]
    bi = 4 * sh.N * sh.C * sh.Hin * sh.Win
    bo = 4 * sh.N * sh.K * sh.H * sh.W
    print(json.dumps({"copies": copies(bi, bo), "in_bytes": bi, "out_bytes": bo}), flush=True)
    for c in ["", "2", "3", "4", "6", "8", "12", "16"]:
        env = dict(os.environ)
        if c:
            env["CONV_HOST_CHUNKS"] = c
        r = subprocess.run([sys.executable, __file__, "--one", path, cfg], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr.strip()[-300:], flush=True)


def copy_pipeline(bi, bo, chunks, n=10):
    """H2D of chunk j on one stream, D2H of chunk j (after its H2D) on another:
    the copy-only floor of conv_run_host's pipeline."""
    dev = torch.device("cuda", 0)
    hi = torch.empty(bi // 4, dtype=torch.float32).pin_memory()
    ho = torch.empty(bo // 4, dtype=torch.float32).pin_memory()
    di = torch.empty(bi // 4, dtype=torch.float32, device=dev)
    do = torch.empty(bo // 4, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    ib = [bi // 4 * j // chunks for j in range(chunks + 1)]
    ob = [bo // 4 * j // chunks for j in range(chunks + 1)]

    def step():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for j in range(chunks):
            with torch.cuda.stream(s1):
                di[ib[j]:ib[j + 1]].copy_(hi[ib[j]:ib[j + 1]], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                ho[ob[j]:ob[j + 1]].copy_(do[ob[j]:ob[j + 1]], non_blocking=True)
        cur.wait_stream(s2)
        cur.wait_stream(s1)
    step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    for _ in range(n):
        step()
    b.record(cur)
    torch.cuda.synchronize()
    return {"copy_pipeline_chunks": chunks, "ms": round(a.elapsed_time(b) / n, 4)}


if __name__ == "__main__" and os.environ.get("PROBE_COPY_PIPELINE"):
    from paper_2101_09808_b200.inputs import CONFIGS
    sh = CONFIGS["batched"]
    for c in (1, 2, 4, 6, 8, 16):
        print(json.dumps(copy_pipeline(4 * sh.N * sh.C * sh.Hin * sh.Win, 4 * sh.N * sh.K * sh.H * sh.W, c)), flush=True)


def copies_under_load(path="fp32_simt", reps=5):
    """The copy pipeline (16 chunks) alone and while the batched layer's
    conv_run (path) runs back to back on another stream."""
    from paper_2101_09808_b200 import conv
    from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
    sh = CONFIGS["batched"]
    xi, wi = make_inputs(sh, seed=0)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path)
    i, k = xi.cuda(), wi.cuda()
    o, ws = plan.new_output(), plan.new_workspace()
    bi, bo = 4 * sh.N * sh.C * sh.Hin * sh.Win, 4 * sh.N * sh.K * sh.H * sh.W
    alone = copy_pipeline(bi, bo, 16)
    s = torch.cuda.Stream()
    res = []
    for _ in range(reps):
        with torch.cuda.stream(s):
            for _ in range(8):
                plan.run(i, k, o, ws, stream=s)
        res.append(copy_pipeline(bi, bo, 16, n=3)["ms"])
        torch.cuda.synchronize()
    return {"alone_ms": alone["ms"], "under_load_ms": res}


if __name__ == "__main__" and os.environ.get("PROBE_COPY_LOAD"):
    print(json.dumps(copies_under_load(os.environ.get("PROBE_COPY_LOAD"))), flush=True)


def overlap_test(path="fp32_simt", chunks=16, reps=3):
    """Is the link slower while conv kernels run?  All work on explicit
    non-blocking streams; timing events on the copy streams themselves.
    Reports the 16-chunk H2D+D2H pipeline alone, then with a chain of conv
    kernels launched first on another stream (and the chain's own span)."""
    from paper_2101_09808_b200 import conv
    from paper_2101_09808_b200.inputs import CONFIGS, make_inputs
    sh = CONFIGS["batched"]
    xi, wi = make_inputs(sh, seed=0)
    plan = conv.ConvPlan(*sh.as_tuple(), path=path)
    i, k = xi.cuda(), wi.cuda()
    o, ws = plan.new_output(), plan.new_workspace()
    bi, bo = 4 * sh.N * sh.C * sh.Hin * sh.Win, 4 * sh.N * sh.K * sh.H * sh.W
    dev = torch.device("cuda", 0)
    hi = torch.empty(bi // 4, dtype=torch.float32).pin_memory()
    ho = torch.empty(bo // 4, dtype=torch.float32).pin_memory()
    di = torch.empty(bi // 4, dtype=torch.float32, device=dev)
    do = torch.empty(bo // 4, dtype=torch.float32, device=dev)
    s1, s2, sk = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
    ib = [bi // 4 * j // chunks for j in range(chunks + 1)]
    ob = [bo // 4 * j // chunks for j in range(chunks + 1)]

    def pipeline():
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s1)
        s2.wait_event(a)
        for j in range(chunks):
            with torch.cuda.stream(s1):
                di[ib[j]:ib[j + 1]].copy_(hi[ib[j]:ib[j + 1]], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                ho[ob[j]:ob[j + 1]].copy_(do[ob[j]:ob[j + 1]], non_blocking=True)
        s1.wait_stream(s2)
        b.record(s1)
        return a, b

    out = {"alone": [], "loaded": [], "kernel_span": []}
    for _ in range(reps):
        a, b = pipeline()
        torch.cuda.synchronize()
        out["alone"].append(round(a.elapsed_time(b), 4))
    for _ in range(reps):
        ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ka.record(sk)
        with torch.cuda.stream(sk):
            for _ in range(6):
                plan.run(i, k, o, ws, stream=sk)
        kb.record(sk)
        a, b = pipeline()
        torch.cuda.synchronize()
        out["loaded"].append(round(a.elapsed_time(b), 4))
        out["kernel_span"].append(round(ka.elapsed_time(kb), 4))
        out.setdefault("copy_start_after_kernels_start", []).append(round(ka.elapsed_time(a), 4))
    # the kernels read the very buffer the uploads write (and write the one
    # the downloads read), as in conv_run_host (a race; timing only)
    di4, do4 = di.view(sh.in_shape), do.view(sh.out_shape)
    for _ in range(reps):
        ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ka.record(sk)
        with torch.cuda.stream(sk):
            for _ in range(6):
                plan.run(di4, k, do4, ws, stream=sk)
        kb.record(sk)
        a, b = pipeline()
        torch.cuda.synchronize()
        out.setdefault("loaded_same_buffers", []).append(round(a.elapsed_time(b), 4))
    return out


if __name__ == "__main__" and os.environ.get("PROBE_OVERLAP"):
    print(json.dumps(overlap_test(os.environ.get("PROBE_OVERLAP"))), flush=True)
