"""Debug build (-DMA_VERIFY): run the table1-shaped sequence with two fused solvers and report which
fused-phase outputs differ from the 5-kernel recomputation, and where."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

NAMES = ["z", "p", "v", "s", "zs", "t", "slots"]
dates = int(sys.argv[1]) if len(sys.argv) > 1 else 22
base = gen.CONFIGS["C4"].with_(cv=(5.0, 20.0), dl=(1e-4, 1e-3))
g = (base.nx, base.ny, base.nz)
nx, nz = base.nx, base.nz
strips = min(base.ny, 148 // ((nx + 127) // 128))
L = egs.lib()
L.eg_debug_verify.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
cnt = (ctypes.c_ulonglong * 8)()
rec = (ctypes.c_longlong * 256)()
nrec = ctypes.c_int()
st = torch.cuda.Stream()
tot = 0
with torch.cuda.stream(st):
    bands = torch.empty((7, base.n), dtype=torch.float64, device="cuda")
    b = torch.empty(base.n, dtype=torch.float64, device="cuda")
    x = torch.empty(base.n, dtype=torch.float64, device="cuda")
    gen.device(base, bands, b, stream=st)
    sv = [egs.Solver(g, bands, "mixed", stream=st) for _ in range(2)]
    L.eg_debug_verify(cnt, rec, ctypes.byref(nrec))
    for d in range(dates):
        gen.device(base.with_(seed=4 + d % 11), bands, b, stream=st)
        for si, s in enumerate(sv):
            for tol in (1e-3, 1e-4):
                s.set_operator(bands)
                _, info, _ = s.solve(b, tol=tol, maxit=200, out=x)
                L.eg_debug_verify(cnt, rec, ctypes.byref(nrec))
                if any(cnt[i] for i in range(7)):
                    tot += 1
                    print(f"date {d} solver {si} tol {tol:g} ({info.iters} it): mismatches "
                          + ", ".join(f"{NAMES[i]}={cnt[i]}" for i in range(7) if cnt[i]), flush=True)
                    for r in range(min(nrec.value, 12)):
                        import struct
                        idn, q = rec[4 * r], rec[4 * r + 1]
                        va = struct.unpack("d", struct.pack("q", rec[4 * r + 2]))[0]
                        vb = struct.unpack("d", struct.pack("q", rec[4 * r + 3]))[0]
                        if idn == 6:
                            T = (nx + 127) // 128
                            qq, rem = divmod(q, base.ny * T)
                            print(f"   slots[{q}] quantity {qq} row {rem // T} tile {rem % T}: fused {va!r} 5-kernel {vb!r}")
                            continue
                        j, rem = divmod(q, nx * nz)
                        k, i = divmod(rem, nx)
                        rps = base.ny / strips
                        stp = int(j // rps)
                        print(f"   {NAMES[idn]} row {j} (strip {stp}, rows {int(stp * rps)}..{int((stp + 1) * rps) - 1}) "
                              f"level {k} col {i} (tile {i // 128}, lane {i % 128}): fused {va!r} 5-kernel {vb!r}")
print(f"{tot} solves with mismatching fused-phase outputs", flush=True)
