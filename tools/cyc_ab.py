"""Cycle-count A/B of libtagg builds: clock-independent (the GEMM runs power-capped, so wall
time drifts with the SM clock).  Two steps, both on the GPU box:

  ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none \\
      --cache-control none --csv --log-file gpurun_out/cyc.csv python tools/cyc_ab.py A.so B.so -- shapes...
  python tools/cyc_ab.py --report gpurun_out/cyc.csv A.so B.so -- shapes...

Each (shape, library) pair launches REPS times after one warm-up, libraries interleaved;
the report prints the median per pair."""
import csv
import ctypes
import sys

sys.path.insert(0, ".")
REPS = 5


def shapes_table():
    from bench import deepseek_gateup_sizes
    _, local = deepseek_gateup_sizes(seed=0)
    counts, _ = deepseek_gateup_sizes(seed=1)
    q, _ = deepseek_gateup_sizes(seed=2, experts=128, local=128)
    return {
        "ds_gateup": ([local], 4096, 7168, 32, "kn"),
        "ds_down": ([counts], 7168, 2048, 256, "kn"),
        "q_fgu": ([q], 3072, 4096, 128, "kn"),
        "q_fdn": ([q], 4096, 1536, 128, "kn"),
        "q_ddn": ([q], 1536, 4096, 128, "nk"),
        "q_dgu": ([q], 4096, 3072, 128, "nk"),
        "sweep_r64": ([tuple(128 * g + 64 for g in range(8))], 4096, 7168, 8, "kn"),
        "sweep_r1": ([tuple(128 * g + 1 for g in range(8))], 4096, 7168, 8, "kn"),
        "sq8192": ([(8192,)], 8192, 8192, 1, "kn"),
    }


def load(path):
    from paper_2508_16584_b200 import _lib
    L = ctypes.CDLL(path)
    for nm, (r, a) in _lib.SIGNATURES.items():
        if hasattr(L, nm):
            getattr(L, nm).restype, getattr(L, nm).argtypes = r, a
    return L


def main():
    argv = sys.argv[1:]
    report = None
    if argv and argv[0] == "--report":
        report, argv = argv[1], argv[2:]
    i = argv.index("--")
    libs, names = argv[:i], argv[i + 1:]
    if report:
        rows = [r for r in csv.reader(open(report)) if len(r) > 10]
        hdr = rows[0]
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        launches = {}
        for r in rows[1:]:
            if "tagg_gemm" in r[ki]:
                launches.setdefault(r[hdr.index("ID")], {})[r[mi]] = float(r[vi].replace(",", ""))
        seq = [launches[k] for k in sorted(launches, key=int)]
        it = 0
        for sh in names:
            it += len(libs)  # warm-up launches
            per = {lib: [] for lib in libs}
            for _ in range(REPS):
                for lib in libs:
                    per[lib].append((seq[it]["sm__cycles_elapsed.max"], seq[it]["gpu__time_duration.sum"]))
                    it += 1
            base = None
            for lib in libs:
                c, t = sorted(per[lib])[REPS // 2]
                base = base or c
                print(f"{sh:10s} {lib.rsplit('/', 1)[-1]:22s} {c / 1e3:9.1f} kclk ({c / base:6.3f})  {t / 1e3:8.1f} us  "
                      f"{c / t:5.2f} GHz")
        return
    import torch
    from bench import Problem
    dev = torch.device("cuda", 0)
    loaded = [load(p) for p in libs]
    table = shapes_table()
    for name in names:
        sizes, n, k, G, bl = table[name]
        P = Problem(torch, name, sizes, n, k, G, dev, seed=1, b_layout=bl)
        layout = 0 if bl == "kn" else 1

        def run(L):
            rc = L.tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(),
                                         layout, G, P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2),
                                         P.gs[0].data_ptr(), G, n, k, P.out.data_ptr(), n, P.m_alloc, None, None, 0,
                                         torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc

        for L in loaded:
            run(L)
        torch.cuda.synchronize()
        for _ in range(REPS):
            for L in loaded:
                run(L)
                torch.cuda.synchronize()
        del P
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
