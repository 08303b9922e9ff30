"""CPU-side checks of the C ABI: the library builds and loads, exports every function that
include/sacd.h declares, and the ctypes structs match the header.  No compute calls
(no GPU here): sacd_init must fail loudly rather than fall back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2003_03572_b200 import build, sacd
    build.build()
    return sacd.load_library()


def header_functions():
    src = open(os.path.join(ROOT, "include", "sacd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sacd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("sacd_init", "sacd_iterate", "sacd_fit", "sacd_factors", "sacd_free"):
        assert f in fns


def test_every_declared_symbol_is_exported(lib):
    from paper_2003_03572_b200 import sacd
    fns = header_functions()
    for f in fns:
        assert hasattr(lib, f), f
    assert set(fns) == set(sacd.EXPORTS)


def test_exports_via_nm(lib):
    from paper_2003_03572_b200 import sacd
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", sacd.LIB_PATH], capture_output=True, text=True).stdout
    for f in header_functions():
        assert re.search(rf"\bT {f}$", out, re.M), f


def test_options_struct_matches_header(lib):
    from paper_2003_03572_b200 import sacd
    o = sacd.Options()
    lib.sacd_default_options(C.byref(o))
    assert o.struct_size == C.sizeof(sacd.Options) == 88
    assert o.precision == sacd.F64 and o.l_mode == sacd.L_DIAG and o.world_size == 1 and o.use_graph == 1
    sz = (C.c_int32 * 4)()
    assert lib.sacd_abi_sizes(sz) == 0
    assert tuple(sz) == (sacd.ABI_VERSION, C.sizeof(sacd.Options), C.sizeof(sacd.IterStats), C.sizeof(sacd.Info))
    assert C.sizeof(sacd.IterStats) == 4 + 12 + 8 + 8 + 24 + 24 + 24 + 8  # k, branch, f, fit, ti, E, E_changed, ms


def test_sass_is_sm100a(lib):
    import subprocess
    from paper_2003_03572_b200 import sacd
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sacd.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_init_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2003_03572_b200 import sacd
    with pytest.raises(sacd.SacdError) as e:
        sacd.Sacd(np.zeros((1, 3), np.uint32), np.ones(1, np.float32), (2, 2, 2), 2, 1)
    assert e.value.code in (sacd.SACD_ECUDA, sacd.SACD_EINVAL)


def test_bad_arguments_rejected_before_cuda(lib):
    from paper_2003_03572_b200 import sacd
    h = C.c_void_p()
    d = (C.c_int64 * 3)(2, 2, 2)
    assert lib.sacd_init(C.byref(h), None, None, 0, d, 0, 1, None) == sacd.SACD_EINVAL     # rank 0
    assert lib.sacd_init(C.byref(h), None, None, 0, d, 257, 1, None) == sacd.SACD_EINVAL   # rank > 256
    d0 = (C.c_int64 * 3)(0, 2, 2)
    assert lib.sacd_init(C.byref(h), None, None, 0, d0, 2, 1, None) == sacd.SACD_EINVAL    # dim 0
    assert lib.sacd_init(C.byref(h), None, None, -1, d, 2, 1, None) == sacd.SACD_EINVAL    # nnz < 0
    assert b"sacd_init" in lib.sacd_last_error()


def test_variant_without_tuning_build_rejected(lib):
    """The product library carries only the default MTTKRP kernels: a tuning variant is
    EINVAL before any CUDA call (the tuning build is libsacd_tuning.so)."""
    from paper_2003_03572_b200 import sacd
    o = sacd.Options()
    lib.sacd_default_options(C.byref(o))
    o.mttkrp_variant = 39
    h = C.c_void_p()
    d = (C.c_int64 * 3)(2, 2, 2)
    assert lib.sacd_init(C.byref(h), None, None, 0, d, 64, 1, C.byref(o)) == sacd.SACD_EINVAL
    assert b"tuning" in lib.sacd_last_error()


def test_torch_inputs_are_validated(lib):
    """Torch tensors go to the library by data_ptr() without a copy, so the binding refuses
    a dtype / shape / stride the header does not declare instead of reinterpreting it."""
    import torch
    from paper_2003_03572_b200 import sacd
    good_c = torch.zeros((4, 3), dtype=torch.int32)
    good_v = torch.ones(4, dtype=torch.float32)
    bad = [(good_c.to(torch.int64), good_v), (torch.zeros((3, 4), dtype=torch.int32).t(), good_v),
           (torch.zeros((4, 2), dtype=torch.int32), good_v), (good_c, good_v.to(torch.float64)),
           (good_c, torch.ones((4, 1), dtype=torch.float32)), (good_c, torch.ones(8, dtype=torch.float32)[::2]),
           (good_c, torch.ones(5, dtype=torch.float32))]
    for c, v in bad:
        with pytest.raises((TypeError, ValueError)):
            sacd.Sacd(c, v, (2, 2, 2), 2, 1)


def test_build_stamp_is_path_independent_and_taken_before_compile(tmp_path):
    """A prebuilt .so travels to the GPU box into a scratch checkout: its stamp must match
    there (no silent 3-minute rebuild inside the bench or the tests), and an edit made while
    nvcc runs must leave the stamp stale (the stamp is the fingerprint taken before nvcc
    reads the sources)."""
    import importlib.util
    import inspect
    import shutil
    from paper_2003_03572_b200 import build as B
    here = B._fingerprint("default")
    root2 = tmp_path / "elsewhere"
    (root2 / "paper_2003_03572_b200").mkdir(parents=True)
    shutil.copytree(os.path.join(B.ROOT, "include"), root2 / "include")
    shutil.copytree(B.CSRC, root2 / "paper_2003_03572_b200" / "csrc")
    shutil.copy(os.path.join(B.HERE, "build.py"), root2 / "paper_2003_03572_b200" / "build.py")
    spec = importlib.util.spec_from_file_location("build_elsewhere", root2 / "paper_2003_03572_b200" / "build.py")
    B2 = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B2)
    assert B2.ROOT != B.ROOT
    assert B2._fingerprint("default") == here
    assert B2._fingerprint("tuning") != here
    with open(root2 / "paper_2003_03572_b200" / "csrc" / "kernels.cu", "a") as fh:
        fh.write("// edited\n")
    assert B2._fingerprint("default") != here
    src = inspect.getsource(B.build)
    assert src.index("fp = _fingerprint(flavour)") < src.index("subprocess.run(cmd")
