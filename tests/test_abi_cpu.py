"""CPU-side checks of the C ABI library (no GPU needed): it loads, exports every
symbol include/spamm.h declares, and its pure host logic behaves."""
import ctypes
import os
import random

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sp():
    from paper_2103_13042_b200 import build
    build.build()
    from paper_2103_13042_b200 import spamm
    return spamm


def test_library_exports_every_declared_symbol(sp):
    lib = ctypes.CDLL(sp.LIB_PATH)
    declared = sp.declared_functions()
    assert len(declared) >= 20
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing


def test_sm100a_only_cubin(sp):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sp.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", sp.LIB_PATH], capture_output=True,
                          text=True).stdout
    # tcgen05 MMA, TMEM load/store and TMA are present in the product library
    for mnemonic in ("UTCHMMA", "UTCBAR", "LDTM", "UTMALDG"):
        assert mnemonic in sass, mnemonic


def test_status_strings_and_argument_errors(sp):
    assert sp._status_name(0) == "SPAMM_OK"
    assert sp._status_name(6) == "SPAMM_E_STATE"
    for bad_tau in (float("nan"), -1.0, float("inf")):
        with pytest.raises(sp.SpammError) as e:
            sp.spamm_plan(1024, 32, bad_tau, sp.SPAMM_FP32)
        assert e.value.status == sp.SPAMM_E_INVALID
    with pytest.raises(sp.SpammError) as e:
        sp.spamm_plan_ex(0, 4, 4, 32, 1.0, sp.SPAMM_FP32)
    assert e.value.status == sp.SPAMM_E_INVALID
    with pytest.raises(sp.SpammError) as e:
        sp.spamm_plan(64, 48, 1.0, sp.SPAMM_FP32)
    assert e.value.status == sp.SPAMM_E_INVALID


def _load(work, cut):
    return [sum(work[cut[r]:cut[r + 1]]) for r in range(len(cut) - 1)]


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_partition_balanced_by_work(sp, nranks):
    """Sec. 3.5.1 load balance applied to the Sec. 3.4 row partition:
    max_r load_r <= total/nranks + max_i work_i, cuts monotone and covering."""
    rng = random.Random(nranks)
    cases = [
        [10] * 64,                                                         # uniform
        [int(100 * 0.97 ** abs(i - 32)) for i in range(64)],               # banded, light edges
        [1] * 30 + [1000] + [1] * 33,                                      # one heavy row
        [0] * 16,                                                          # no work
        [rng.randint(0, 50) for _ in range(7)],                            # fewer rows than ranks
    ]
    for work in cases:
        cut = sp.spamm_partition_rows(work, nranks)
        assert cut[0] == 0 and cut[-1] == len(work)
        assert all(a <= b for a, b in zip(cut, cut[1:]))
        total = sum(work)
        assert max(_load(work, cut)) <= total / nranks + max(work) + 1e-9


def test_partition_rejects_bad_input(sp):
    with pytest.raises(sp.SpammError):
        sp.spamm_partition_rows([1, -1, 2], 2)
    with pytest.raises(sp.SpammError):
        sp.spamm_partition_rows([1, 2], 0)


def test_product_path_never_touches_the_oracle():
    """The oracle is test infrastructure: the package neither imports it nor shares code with it,
    and importing the binding leaves it unloaded (checked in a fresh interpreter)."""
    import glob
    import subprocess
    import sys
    pkg = os.path.join(ROOT, "paper_2103_13042_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True) + glob.glob(os.path.join(pkg, "csrc", "*")):
        txt = open(f, errors="ignore").read()
        assert "import oracle" not in txt and "from oracle" not in txt, f
    code = ("import sys; sys.path.insert(0, %r); from paper_2103_13042_b200 import spamm; "
            "print('oracle' in sys.modules)" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd="/tmp")
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("False")


def test_binding_refuses_to_load_without_the_library(tmp_path):
    """No fallback: a copy of the binding next to no libspamm.so raises ImportError on import."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_2103_13042_b200"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_2103_13042_b200", "spamm.py"), pkg / "spamm.py")
    (pkg / "__init__.py").write_text("")
    code = "import sys; sys.path.insert(0, %r); from paper_2103_13042_b200 import spamm" % str(tmp_path)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.returncode != 0 and "ImportError" in out.stderr
