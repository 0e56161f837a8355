"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/sqngd.h declares; host-only utilities work without a GPU."""
import ctypes as C
import os
import re

import pytest

from paper_2604_25728_b200 import sqngd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "sqngd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sqngd_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_25728_b200 import build

    build.build()
    return sqngd.lib()


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(sqngd.EXPORTED) == names


def test_struct_layouts():
    # sqngd_metrics: 6 doubles + 8 int32 + 2 uint32 + 4 doubles (PSLR x3, SNRL) = 120 bytes;
    # sqngd_state: 9 pointers + 2 int64 + 4 pointers
    assert sqngd.METRICS_BYTES == 120
    assert C.sizeof(sqngd.State) == 9 * 8 + 16 + 4 * 8


def test_version_and_units(lib):
    assert b"sm_100a" in lib.sqngd_version()
    from paper_2604_25728_b200.configs import C3, C5

    assert lib.sqngd_num_units(C.byref(sqngd.make_config(C3))) == 8 * 257
    assert lib.sqngd_num_units(C.byref(sqngd.make_config(C5))) == 8 * 16 * 513


@pytest.mark.parametrize("units,world", [(2056, 1), (2056, 2), (2056, 8), (7, 8), (65664, 3), (0, 4)])
def test_shard_range_partitions(lib, units, world):
    spans = [sqngd.shard_range(units, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == units
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_create_rejects_invalid_config_without_gpu(lib):
    """Validation happens before any CUDA call, so it is testable on CPU."""
    from paper_2604_25728_b200.configs import C1

    h = C.c_void_p()
    empty_roi = C1.with_(M=1, tau_lo=0, tau_hi=0)      # auto map only, tau = 0 excluded (Eq. 8): no cells
    for bad in (C1.with_(B=1), C1.with_(N=1), C1.with_(K=0), C1.with_(tau_lo=-64), C1.with_(N=8192), empty_roi,
                C1.with_(doppler_engine=3), C1.with_(net_width=12, net_depth=5),
                C1.with_(net_width=256, net_depth=5), C1.with_(net_width=128, net_depth=-1),
                C1.with_(net_width=128, net_depth=40)):
        cfg = sqngd.make_config(bad)
        st = lib.sqngd_create(C.byref(cfg), 0, None, 0, 1, C.byref(h))
        assert st == sqngd.E_INVALID
        assert lib.sqngd_last_error(None)


def test_peer_api_rejects_null_arguments_without_gpu(lib):
    """The peer-memory all-reduce entry points (include/sqngd.h sqngd_peer_export / _attach,
    sqngd_loopback_set_peer) check their arguments before any CUDA call."""
    buf = C.create_string_buffer(64)
    assert lib.sqngd_peer_export(None, buf) == sqngd.E_INVALID
    assert lib.sqngd_peer_attach(None, buf) == sqngd.E_INVALID
    assert lib.sqngd_loopback_set_peer(None, 1) == sqngd.E_INVALID
    assert b"null" in lib.sqngd_last_error(None)


def test_generator_parameter_count(lib):
    """sqngd_net_num_params = the closed form D (2 W^2 + 2 W) + (W Din + W) + (Din W + Din)."""
    from paper_2604_25728_b200.configs import C1, C3

    assert sqngd.net_num_params(C3) == 0
    for c, W, D in ((C3, 128, 5), (C1, 32, 2), (C1.with_(M=3, N=37), 8, 0)):
        Din = c.M * c.N
        n = D * (2 * W * W + 2 * W) + 2 * W * Din + W + Din
        assert sqngd.net_num_params(c.with_(net_width=W, net_depth=D)) == (n + 3) // 4 * 4  # float4 stride
