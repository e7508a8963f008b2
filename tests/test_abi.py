"""CPU-side checks of the C-ABI library: it builds, loads, and exports every
symbol include/rgnn.h declares; argument errors come back as status codes
(no compute call is made without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rgnn.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"RGNN_API\s+[\w\s\*]+?\b(rgnn_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2412_04747_b200 import build
    build.build()
    from paper_2412_04747_b200 import rgnn
    return rgnn.lib()


def test_header_declares_api():
    syms = declared_symbols()
    assert "rgnn_graph_build" in syms and "rgnn_layer_backward" in syms and len(syms) >= 14


def test_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
    from paper_2412_04747_b200 import rgnn
    assert sorted(rgnn.EXPORTED) == declared_symbols()


def test_version_and_error_paths(lib):
    from paper_2412_04747_b200 import rgnn
    assert "sm_100a" in rgnn.version()
    # NULL arguments -> INVALID_ARG with a message, never a crash
    assert lib.rgnn_layer_workspace(None, None, None, None) == 1
    assert "NULL" in lib.rgnn_last_error().decode()
    out = C.c_void_p()
    ntp = (C.c_int64 * 2)(0, 4)
    st = lib.rgnn_graph_build(4, 1, ntp, 0, 0, None, None, None, 0, 4, rgnn.ALLOC_FN(0), rgnn.FREE_FN(0), None,
                              None, C.byref(out))
    assert st == 1 and "num_rels" in lib.rgnn_last_error().decode()
    ntp_bad = (C.c_int64 * 2)(0, 3)
    st = lib.rgnn_graph_build(4, 1, ntp_bad, 1, 0, None, None, None, 0, 4, rgnn.ALLOC_FN(0), rgnn.FREE_FN(0), None,
                              None, C.byref(out))
    assert st == 1 and "node_type_ptr" in lib.rgnn_last_error().decode()
    assert lib.rgnn_graph_destroy(None) == 0


def test_sass_is_sm100a(lib):
    import subprocess
    from paper_2412_04747_b200.rgnn import LIB_PATH
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    assert r.returncode == 0
    assert "sm_100a" in r.stdout


def test_segment_plan_argument_errors(lib):
    """rgnn_segment_plan_create validates seg_ptr on the host before touching the device."""
    from paper_2412_04747_b200 import rgnn
    out = C.c_void_p()
    bad = (C.c_int64 * 3)(0, 5, 3)
    st = lib.rgnn_segment_plan_create(2, bad, None, rgnn.ALLOC_FN(0), rgnn.FREE_FN(0), None, None, C.byref(out))
    assert st == 1 and "decreases at segment 1" in lib.rgnn_last_error().decode()
    nz = (C.c_int64 * 2)(1, 5)
    st = lib.rgnn_segment_plan_create(1, nz, None, rgnn.ALLOC_FN(0), rgnn.FREE_FN(0), None, None, C.byref(out))
    assert st == 1 and "seg_ptr[0]" in lib.rgnn_last_error().decode()
    ok = (C.c_int64 * 2)(0, 5)
    negw = (C.c_int32 * 1)(-1)
    st = lib.rgnn_segment_plan_create(1, ok, negw, rgnn.ALLOC_FN(0), rgnn.FREE_FN(0), None, None, C.byref(out))
    assert st == 1 and "negative weight" in lib.rgnn_last_error().decode()
    assert lib.rgnn_segment_gemm(None, 1, None, None, 64, None, 1, 64, 0, None, 1, None, 0, None) == 1
    assert lib.rgnn_segment_plan_destroy(None) == 0


def test_comm_argument_errors(lib):
    """Communicator entry points validate their arguments before touching NCCL or a device."""
    from paper_2412_04747_b200 import rgnn
    out = C.c_void_p()
    ptr = (C.c_int64 * 3)(0, 5, 10)
    uid = C.create_string_buffer(rgnn.COMM_ID_BYTES)
    assert lib.rgnn_comm_create(2, 2, uid, ptr, C.byref(out)) == 1          # rank outside [0, world)
    assert "rank" in lib.rgnn_last_error().decode()
    bad = (C.c_int64 * 3)(0, 6, 5)
    assert lib.rgnn_comm_create(0, 2, uid, bad, C.byref(out)) == 1          # decreasing node_ptr
    assert lib.rgnn_comm_create(0, 2, None, ptr, C.byref(out)) == 1
    assert lib.rgnn_comm_destroy(None) == 0


def test_exchange_bytes():
    """Variant X moves N d_in b bytes, variant P U_global k d_out b (k = 2 for HGT's [K~|M])."""
    from paper_2412_04747_b200 import rgnn
    e = rgnn.exchange_bytes("hgt", "bf16", 64, 64, num_nodes=1000, num_pairs_global=3000)
    assert e == {"bytes_x": 1000 * 64 * 2, "bytes_p": 3000 * 2 * 64 * 2, "variant": "X"}
    e = rgnn.exchange_bytes("rgcn", "f32", 64, 64, num_nodes=1000, num_pairs_global=3000)
    assert e["bytes_p"] == 3000 * 64 * 4
