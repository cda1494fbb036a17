"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol include/egsolve.h
declares, and its host-only entry points behave (no GPU compute is called here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def egs():
    subprocess.check_call(["make", "-s", "paper_1811_03852_b200/libegsolve.so"], cwd=ROOT,
                          stdout=subprocess.DEVNULL)
    import paper_1811_03852_b200 as m
    return m


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "egsolve.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eg_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared_symbols()
    for f in ("eg_solver_create", "eg_apply_operator", "eg_precondition", "eg_solve"):
        assert f in names


def test_library_exports_every_declared_symbol(egs):
    L = egs.lib()
    for name in _declared_symbols():
        assert hasattr(L, name), name
    assert set(egs.ABI_SYMBOLS) == set(_declared_symbols())


def test_status_strings_and_kernel_names(egs):
    L = egs.lib()
    for code, name in egs.STATUS.items():
        assert L.eg_status_str(code).decode() == name
    names = [L.eg_kernel_name(k).decode() for k in range(L.eg_num_kernels())]
    assert {"thomas_p", "stencil_dot_A", "thomas_s", "stencil_dot_B", "update_xr"} <= set(names)


def test_workspace_bytes_and_argument_validation(egs):
    L = egs.lib()
    g = egs._Grid(2560, 1920, 70)
    nb = ctypes.c_size_t()
    assert L.eg_workspace_bytes(ctypes.byref(g), None, egs.EG_MIXED, ctypes.byref(nb)) == 0
    n = 2560 * 1920 * 70
    # 6 fp32 bands + diag + bhat + x(fp64) + 8 fp32 vectors: the MIXED footprint
    assert 6 * 4 * n + 3 * 8 * n + 8 * 4 * n <= nb.value <= 6 * 4 * n + 3 * 8 * n + 8 * 4 * n + 64 * 2**20
    nb64 = ctypes.c_size_t()
    assert L.eg_workspace_bytes(ctypes.byref(g), None, egs.EG_FP64, ctypes.byref(nb64)) == 0
    assert nb64.value > nb.value
    bad = egs._Grid(2, 10, 10)          # nx < 3 (reading A-19)
    assert L.eg_workspace_bytes(ctypes.byref(bad), None, egs.EG_MIXED, ctypes.byref(nb)) == 1
    for dims in ((8, 0, 4), (8, 4, 0), (-8, 4, 4), (1 << 26, 4, 64)):   # empty grids; nx*nz >= 2^31
        bad = egs._Grid(*dims)
        assert L.eg_workspace_bytes(ctypes.byref(bad), None, egs.EG_MIXED, ctypes.byref(nb)) == 1, dims
    assert L.eg_workspace_bytes(ctypes.byref(g), None, 3, ctypes.byref(nb)) == 1     # unknown precision
    # decomposition must align with the 8 reduction row-groups
    d = egs._Dist(0, 960, 0, 2, None)
    assert L.eg_workspace_bytes(ctypes.byref(g), ctypes.byref(d), egs.EG_MIXED, ctypes.byref(nb)) == 0
    d = egs._Dist(0, 961, 0, 2, None)
    assert L.eg_workspace_bytes(ctypes.byref(g), ctypes.byref(d), egs.EG_MIXED, ctypes.byref(nb)) == 1
    d = egs._Dist(0, 640, 0, 3, None)    # 3 does not divide 8
    assert L.eg_workspace_bytes(ctypes.byref(g), ctypes.byref(d), egs.EG_MIXED, ctypes.byref(nb)) == 1
    # EG_FEATURE_TRISOR: + colour-split (E,W,N,S), (U,D), f and the sweeps' x (ghosted: + 2 rows),
    # 8 working-precision values per point
    assert L.eg_workspace_bytes(ctypes.byref(g), None, egs.EG_MIXED, ctypes.byref(nb)) == 0
    nbt, nb0 = ctypes.c_size_t(), ctypes.c_size_t()
    assert L.eg_workspace_bytes_ex(ctypes.byref(g), None, egs.EG_MIXED, 0, ctypes.byref(nb0)) == 0
    assert nb0.value == nb.value
    assert L.eg_workspace_bytes_ex(ctypes.byref(g), None, egs.EG_MIXED, egs.EG_FEATURE_TRISOR, ctypes.byref(nbt)) == 0
    row = g.nx * g.nz
    assert (8 * n + 2 * row) * 4 <= nbt.value - nb.value <= (8 * n + 2 * row) * 4 + 256
    assert L.eg_workspace_bytes_ex(ctypes.byref(g), None, egs.EG_MIXED, 4, ctypes.byref(nbt)) == 1  # unknown bit
    h = ctypes.c_void_p()
    assert L.eg_solver_create(None, None, None, 1, None, 0, None, ctypes.byref(h)) == 1
    assert not h.value
    bands = (ctypes.c_void_p * 7)(*([1] * 7))
    ws = ctypes.c_void_p(256)
    # eg_solver_create_ex: an unknown feature bit is refused before any device work
    assert L.eg_solver_create_ex(ctypes.byref(g), None, bands, 1, 4, ws, nbt.value, None, ctypes.byref(h)) == 1
    assert not h.value


def test_band_rows_partition(egs):
    for ny in (48, 144, 480, 1152, 1920, 37, 5):
        G = min(8, ny)
        for P in (1, 2, 4, 8):
            if G % P:
                with pytest.raises(ValueError):
                    egs.band_rows(ny, 0, P)
                continue
            rows = [egs.band_rows(ny, r, P) for r in range(P)]
            assert rows[0][0] == 0 and rows[-1][1] == ny
            assert all(rows[r][1] == rows[r + 1][0] for r in range(P - 1))
            assert all(b > a for a, b in rows)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1811_03852_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "liboracle" not in txt


def test_transport_codes_match_the_header(egs):
    """eg_solver_transport's EG_TRANSPORT_* codes (include/egsolve.h) are the names the binding's
    Solver.transport reports, and a NULL handle is an argument error."""
    src = open(os.path.join(ROOT, "include", "egsolve.h")).read()
    codes = {int(v): k for k, v in re.findall(r"#define EG_TRANSPORT_([A-Z0-9_]+)\s+(\d+)", src)}
    assert codes == {0: "NONE", 1: "NCCL", 2: "P2P", 3: "LOOPBACK", 4: "LOOPBACK_P2P"}
    assert {k: v.lower().replace("_", "-") for k, v in codes.items()} == egs.Solver.TRANSPORTS
    assert egs.lib().eg_solver_transport(None) < 0
    # the IPC test hooks reject NULL arguments without touching the GPU
    rec = ctypes.create_string_buffer(80)
    assert egs.lib().eg_debug_ipc_export(None, rec) == 1
    p, o = ctypes.c_void_p(), ctypes.c_void_p()
    assert egs.lib().eg_debug_ipc_open(None, ctypes.byref(p), ctypes.byref(o)) == 1
