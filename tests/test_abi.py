"""CPU-side checks of the C ABI: libsonic.so builds, loads without a GPU, exports every
function include/sonic.h declares, and its host-side logic (sizes, validation) behaves.
No compute call is made here (there is no GPU in CI)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sonic.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2512_14080_b200 import build, sonic
    build.build()
    return sonic.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*[A-Za-z_][\w\s\*]*?\b(sonic_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("sonic_route", "sonic_moe_fwd", "sonic_moe_bwd", "sonic_rows_max", "sonic_routing_sizes",
                 "sonic_route_workspace_size", "sonic_fwd_workspace_size", "sonic_bwd_workspace_size",
                 "sonic_status_string"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), f"libsonic.so does not export {name}"


def test_host_side_sizes(lib):
    from paper_2512_14080_b200 import sonic
    from paper_2512_14080_b200.inputs import CONFIGS
    for name, c in CONFIGS.items():
        for mode in (sonic.SONIC_ROUTE_TC, sonic.SONIC_ROUTE_TR_NRF):
            d = sonic.make_desc(c["T"], c["d"], c["n"], c["E"], c["K"], mode=mode)
            rows = sonic.sonic_rows_max(d)
            TK = c["T"] * c["K"]
            assert rows % 128 == 0 and TK <= rows <= TK + c["E"] * 127 + 127
            sz = sonic.sonic_routing_sizes(d)
            assert sz["row_token"] == rows * 4 and sz["topk_ids"] == TK * 4
            assert sz["token_rowptr"] == (c["T"] + 1) * 4
            assert sonic.sonic_route_workspace_size(d) > 0
            # fwd workspace holds Y [rows,d] and A [rows,n] in bf16; with the opt-in fused up/down
            # kernel (n = 128 / 256, d % 128 == 0) A stays on chip: Y only
            assert sonic.sonic_fwd_workspace_size(d) >= rows * (c["n"] + c["d"]) * 2
            if c["n"] in (128, 256) and c["d"] % 128 == 0:
                df = sonic.make_desc(c["T"], c["d"], c["n"], c["E"], c["K"], mode=mode,
                                     flags=sonic.SONIC_F_FUSED_UPDOWN)
                assert rows * c["d"] * 2 <= sonic.sonic_fwd_workspace_size(df) < rows * (c["n"] + c["d"]) * 2
            assert sonic.sonic_bwd_workspace_size(d) >= rows * (3 * c["n"] + c["d"]) * 2


@pytest.mark.parametrize("T,E,K", [(4097, 256, 8), (8193, 256, 8), (16385, 256, 8), (300, 200, 6), (100, 1, 1),
                                   (4096, 128, 8)])
def test_ec_rows_bound_covers_capacity(lib, T, E, K):
    """Expert choice keeps C = min(ceil_M(ceil(T K / E)), T) rows per expert (Q22); rows_max must hold
    E tiles-rounded copies of C (E*C can exceed T K + E*127 once E > 128)."""
    from paper_2512_14080_b200 import sonic
    for m_tile in (128, 256):
        d = sonic.make_desc(T, 128, 64, E, K, mode=sonic.SONIC_ROUTE_EC, m_tile=m_tile)
        C = min(-(-(-(-T * K // E)) // m_tile) * m_tile, T)
        need = E * (-(-C // 128) * 128)
        assert sonic.sonic_rows_max(d) >= need


def test_invalid_arguments_are_rejected_before_any_launch(lib):
    from paper_2512_14080_b200 import sonic
    bad = [
        sonic.make_desc(256, 64, 32, 8, 9),        # K > E
        sonic.make_desc(256, 64, 32, 8, 0),        # K = 0
        sonic.make_desc(256, 64, 32, 5000, 2),     # E > 4096
        sonic.make_desc(256, 64, 32, 8, 17),       # K > 16
        sonic.make_desc(256, 64, 32, 8, 2, m_tile=64),
        sonic.make_desc(0, 64, 32, 8, 2),
    ]
    for d in bad:
        assert lib.sonic_rows_max(ctypes.byref(d)) == -1
        st = lib.sonic_route(ctypes.byref(d), None, None, None, 0, None)
        assert st == -1, sonic.lib().sonic_status_string(st)
    d = sonic.make_desc(256, 64, 32, 8, 2)
    # null pointers -> INVALID_ARG, no CUDA call is made
    assert lib.sonic_moe_fwd(ctypes.byref(d), None, None, None, None, None, None, None, 0, None) == -1
    assert lib.sonic_moe_bwd(ctypes.byref(d), *([None] * 11), 0, None) == -1
    # unsupported dims -> UNSUPPORTED (d not a multiple of 64)
    d2 = sonic.make_desc(256, 96, 32, 8, 2)
    rt = sonic.sonic_routing(*([1 << 20] * len(sonic.ROUTING_FIELDS)))
    assert lib.sonic_route(ctypes.byref(d2), ctypes.c_void_p(1 << 20), ctypes.byref(rt), None, 0, None) == -2
    # short workspace -> WORKSPACE
    assert lib.sonic_route(ctypes.byref(d), ctypes.c_void_p(1 << 20), ctypes.byref(rt), ctypes.c_void_p(1 << 20), 1,
                           None) == -3
    for s in (0, -1, -2, -3, -4, -5):
        assert lib.sonic_status_string(s)


def test_round2_calls_validate_on_the_host(lib):
    """The round-2 entry points reject bad arguments before any CUDA call (so on a CPU host too)."""
    from paper_2512_14080_b200 import sonic
    P = ctypes.c_void_p(1 << 20)
    rt = sonic.sonic_routing(*([1 << 20] * len(sonic.ROUTING_FIELDS)))
    d = sonic.make_desc(256, 64, 32, 8, 2)
    dg = sonic.make_desc(256, 64, 32, 8, 8, mode=sonic.SONIC_ROUTE_GIVEN)
    # fused softmax: null logits, GIVEN routing, misaligned logits
    assert lib.sonic_route_logits(ctypes.byref(d), None, P, ctypes.byref(rt), P, 1 << 30, None) == -1
    assert lib.sonic_route_logits(ctypes.byref(dg), P, P, ctypes.byref(rt), P, 1 << 30, None) == -1
    assert lib.sonic_route_logits(ctypes.byref(d), ctypes.c_void_p((1 << 20) + 4), P, ctypes.byref(rt), P,
                                  1 << 30, None) == -1
    # capped GIVEN routing: not GIVEN, or no flag
    flag = ctypes.c_void_p(1 << 21)
    assert lib.sonic_route_given_capped(ctypes.byref(d), P, ctypes.byref(rt), P, 1 << 30, flag, None) == -1
    assert lib.sonic_route_given_capped(ctypes.byref(dg), P, ctypes.byref(rt), P, 1 << 30, None, None) == -1
    # router GEMMs: null operands; both outputs null; short workspace
    assert lib.sonic_router_fwd(ctypes.byref(d), None, P, P, None) == -1
    assert lib.sonic_router_grad(ctypes.byref(d), P, P, P, None, None, P, 1 << 30, None) == -1
    assert lib.sonic_router_grad(ctypes.byref(d), P, P, P, P, P, P, 1, None) == -3
    assert lib.sonic_router_grad_workspace_size(ctypes.byref(d)) == 256 * 8 * 2
    # e4m3 quantisers: cols not a multiple of 8, misaligned, null
    assert lib.sonic_quantize_e4m3_rows(P, 10, 12, P, P, None) == -1
    assert lib.sonic_quantize_e4m3_rows(ctypes.c_void_p((1 << 20) + 2), 10, 16, P, P, None) == -1
    assert lib.sonic_quantize_e4m3_cols(None, 1, 16, 16, P, P, None) == -1
    assert lib.sonic_quantize_e4m3_cols(P, 1, 16, 12, P, P, None) == -1
    # FP8 up-projection: n % 128 != 0 -> UNSUPPORTED (checked before the workspace)
    d8 = sonic.make_desc(256, 128, 64, 8, 2, flags=sonic.SONIC_F_FP8_UP)
    assert lib.sonic_moe_fwd(ctypes.byref(d8), P, P, P, ctypes.byref(rt), P, P, P, 1 << 40, None) == -2
    # the fp8 workspace holds the e4m3 copies: bigger than the bf16 one
    d8ok = sonic.make_desc(256, 128, 128, 8, 2, flags=sonic.SONIC_F_FP8_UP)
    d16 = sonic.make_desc(256, 128, 128, 8, 2)
    assert lib.sonic_fwd_workspace_size(ctypes.byref(d8ok)) >= (lib.sonic_fwd_workspace_size(ctypes.byref(d16)) +
                                                                256 * 128 + 8 * 128 * 256)
    # FP8 dX~: d % 256 != 0 -> UNSUPPORTED; with SONIC_F_BWD_DW_ONLY (no dX~ to compute) -> INVALID_ARG;
    # the bwd workspace then holds the e4m3 dH' rows, their scales and W1's e4m3 copy + column scales
    dx8 = sonic.make_desc(256, 128, 128, 8, 2, flags=sonic.SONIC_F_FP8_DXT)
    assert lib.sonic_moe_bwd(ctypes.byref(dx8), P, P, P, P, P, ctypes.byref(rt), P, P, P, P, P, 1 << 40, None) == -2
    dx8ok = sonic.make_desc(256, 256, 128, 8, 2, flags=sonic.SONIC_F_FP8_DXT)
    dx8dw = sonic.make_desc(256, 256, 128, 8, 2, flags=sonic.SONIC_F_FP8_DXT | sonic.SONIC_F_BWD_DW_ONLY)
    assert lib.sonic_moe_bwd(ctypes.byref(dx8dw), P, P, P, P, P, ctypes.byref(rt), P, P, P, P, P, 1 << 40, None) == -1
    d16b = sonic.make_desc(256, 256, 128, 8, 2)
    rows = lib.sonic_rows_max(ctypes.byref(dx8ok))
    assert lib.sonic_bwd_workspace_size(ctypes.byref(dx8ok)) >= (lib.sonic_bwd_workspace_size(ctypes.byref(d16b)) +
                                                                 rows * 256 + rows * 4 + 8 * 256 * 256 + 8 * 256 * 4)
    offs = (ctypes.c_size_t * 4)()
    assert lib.sonic_workspace_offsets(ctypes.byref(dx8ok), 2, offs) == 0 and offs[0] != (1 << 64) - 1
    assert lib.sonic_workspace_offsets(ctypes.byref(d16b), 2, offs) == 0 and offs[0] == (1 << 64) - 1


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2512_14080_b200 import sonic
    monkeypatch.setattr(sonic, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(sonic, "_lib", None)
    with pytest.raises(sonic.SonicError):
        sonic.lib()


def test_m_tile_256_rows_bound(lib):
    """m_tile 256 is accepted and widens the rows bound to E*255 of rounding slack; 64 is rejected."""
    from paper_2512_14080_b200 import sonic
    d = sonic.make_desc(32768, 1536, 256, 128, 8, mode=sonic.SONIC_ROUTE_TR_NRF, m_tile=256)
    assert sonic.sonic_rows_max(d) == (32768 * 8 + 128 * 255 + 127) // 128 * 128
    assert sonic.sonic_rows_max(sonic.make_desc(256, 64, 32, 8, 2, m_tile=64)) == -1


def test_given_rows_cap(lib):
    """SONIC_ROUTE_GIVEN with rows_cap: rows_max = round_128(rows_cap + E*127) (capped by the T*K
    bound); rows_cap on another mode, or negative, is rejected."""
    from paper_2512_14080_b200 import sonic
    d = sonic.make_desc(1000, 64, 64, 32, 32, mode=sonic.SONIC_ROUTE_GIVEN, rows_cap=5000)
    assert sonic.sonic_rows_max(d) == (5000 + 32 * 127 + 127) // 128 * 128
    d0 = sonic.make_desc(1000, 64, 64, 32, 32, mode=sonic.SONIC_ROUTE_GIVEN)
    assert sonic.sonic_rows_max(d0) == min(1000 * 32 + 32 * 127, 32 * 1024)  # E * ceil_128(T) bound
    assert sonic.sonic_rows_max(d) < sonic.sonic_rows_max(d0)
    assert sonic.sonic_rows_max(sonic.make_desc(1000, 64, 64, 32, 8, rows_cap=5000)) == -1
    assert sonic.sonic_rows_max(sonic.make_desc(1000, 64, 64, 32, 32, mode=sonic.SONIC_ROUTE_GIVEN,
                                                rows_cap=-1)) == -1
