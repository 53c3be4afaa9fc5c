"""Host-side drop-in modules against the reference build (oracle/_ref):
perf_model.hpp (Table 1 integers, predictions, profile files), theory.hpp
(rates, spectrum_of), the Matrix Market / block-vector text formats
(sparse_matrix.hpp:133-205, block_vector.hpp:72-112) in C++ (tests/cpp
test_host) and Python (textio.py), and blockkrylov-cli's host-only paths
(model, verify --suite rates, usage / file errors and exit codes,
blockkrylov_cli.cpp:20-24).  No GPU."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import paper_1912_11930_b200 as bk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1912_11930_b200", "_build", "blockkrylov-cli")
HOST = os.path.join(ROOT, "tests", "cpp", "bin", "test_host")
KERNELS = {"bdot": 0, "baxpy": 1, "bop": 2}
BOUND = {0: "compute", 1: "memory", 2: "register"}
SKYLAKE = (76.8e9, 13.345e9, 286.1e9, 8.0)


def run(*args, **kw):
    return subprocess.run(list(args), capture_output=True, text=True, timeout=120, **kw)


@pytest.fixture(scope="module")
def rlib(ref):
    L = ref.lib
    u64p = C.POINTER(C.c_uint64)
    dp = C.POINTER(C.c_double)
    L.bkref_characteristics.argtypes = [C.c_int] + [C.c_size_t] * 4 + [u64p]
    L.bkref_characteristics.restype = C.c_int
    L.bkref_predict.argtypes = [C.c_int] + [C.c_size_t] * 4 + [C.c_double] * 4 + [dp, C.POINTER(C.c_int)]
    L.bkref_predict.restype = C.c_int
    L.bkref_rate.argtypes = [C.c_int, C.c_size_t, dp, C.c_size_t, C.c_size_t]
    L.bkref_rate.restype = C.c_double
    L.bkref_spectrum_of.argtypes = [C.c_size_t, u64p, u64p, dp, dp]
    L.bkref_save_matrix_market.argtypes = [C.c_char_p, C.c_size_t, u64p, u64p, dp]
    L.bkref_save_block_vector.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, dp]
    L.bkref_mm_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
    L.bkref_bv_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
    return L


def _p(a, t):
    return np.ascontiguousarray(a).ctypes.data_as(C.POINTER(t))


def _csr(a):
    return (np.ascontiguousarray(a.row_offsets(), dtype=np.uint64),
            np.ascontiguousarray(a.col_indices(), dtype=np.uint64),
            np.ascontiguousarray(a.values(), dtype=np.float64))


MATRICES = [
    lambda: bk.poisson2d(bk.PoissonSpec.heterogeneous(6, 5, 3)),
    lambda: bk.poisson2d(bk.PoissonSpec.constant(4, 7)),
    lambda: bk.stencil(4, 3, 4, 3),
    lambda: bk.SparseMatrix.from_triplets(3, [(0, 0, 2.0), (1, 1, -0.0), (2, 2, 1e-300),
                                             (0, 2, 1.0 / 3), (2, 0, 1.0 / 3)]),
]


# --------------------------------------------------------------- perf model --
@pytest.mark.parametrize("kernel", ["bdot", "baxpy", "bop"])
@pytest.mark.parametrize("n,k,p,z", [(1000, 8, 1, 5000), (1000, 8, 8, 5000), (2097152, 32, 8, 14581760),
                                     (7, 12, 3, 0), (56623104, 64, 16, 395476992)])
def test_characteristics_match_reference(rlib, kernel, n, k, p, z):
    want = np.zeros(3, dtype=np.uint64)
    assert rlib.bkref_characteristics(KERNELS[kernel], n, k, p, z, _p(want, C.c_uint64)) == 0
    out = run(HOST, "chars", kernel, str(n), str(k), str(p), str(z))
    assert out.returncode == 0, out.stderr
    assert [int(v) for v in out.stdout.split()] == want.tolist()


def test_characteristics_reject_bad_width():
    assert run(HOST, "chars", "bdot", "10", "8", "3", "0").returncode == 2
    assert run(HOST, "chars", "bdot", "10", "8", "0", "0").returncode == 2


def _model(*args, env=None):
    return run(CLI, "model", *args, env=env)


def _parse_model(stdout):
    lines = stdout.strip().split("\n")
    assert lines[0] == "p,t_comp,t_mem,t_reg,t,bound"
    return [(int(f[0]), [float(x) for x in f[1:5]], f[5]) for f in (l.split(",") for l in lines[1:])]


@pytest.mark.parametrize("kernel,extra", [("bdot", []), ("baxpy", []), ("bop", ["--z", "77777"])])
@pytest.mark.parametrize("machine", ["default", "b200", "file"])
def test_cli_model_matches_reference_predict(rlib, tmp_path, kernel, extra, machine):
    n, k, ps = 123457, 64, [1, 2, 4, 8, 16, 32, 64]
    args = ["--kernel", kernel, "--n", str(n), "--k", str(k), "--p-list", ",".join(map(str, ps))] + extra
    if machine == "default":
        prof = SKYLAKE
    elif machine == "b200":
        prof = (40.0e12, 6553.3e9, 148.0 * 128.0 * 1.965e9, 8.0)
        args += ["--machine", "b200"]
    else:
        prof = (1e9, 2e9, 3e10, 4.0)
        f = tmp_path / "m.prof"
        f.write_text("# test profile\n\npeak_flops = 1e9\nmem_bandwidth=2e9\n  reg_bandwidth = 3e10\n"
                     "bytes_per_scalar = 4\nunknown_key = 5\n")
        args += ["--machine", str(f)]
    env = dict(os.environ)
    env.pop("BLOCKKRYLOV_MACHINE", None)
    out = _model(*args, env=env)
    assert out.returncode == 0, out.stderr
    rows = _parse_model(out.stdout)
    assert [r[0] for r in rows] == ps
    z = int(extra[1]) if extra else 0
    for p, t, bound in rows:
        want = np.zeros(4)
        b = C.c_int()
        assert rlib.bkref_predict(KERNELS[kernel], n, k, p, z, *prof, _p(want, C.c_double), C.byref(b)) == 0
        assert t == want.tolist()  # %.17g round-trips exactly
        assert bound == BOUND[b.value]


def test_cli_model_machine_from_environment(tmp_path):
    f = tmp_path / "env.prof"
    f.write_text("peak_flops=1\nmem_bandwidth=1\nreg_bandwidth=1\n")
    env = dict(os.environ, BLOCKKRYLOV_MACHINE=str(f))
    out = _model("--kernel", "bdot", "--n", "10", "--k", "2", "--p-list", "1", env=env)
    assert out.returncode == 0
    p, t, bound = _parse_model(out.stdout)[0]
    # omega = 2*10*1*2 = 40 flop, beta = 40 scalars, tau = 2*10*2 + 40 = 80 scalars
    assert t[:3] == [40.0, 320.0, 640.0] and bound == "register"


@pytest.mark.parametrize("args,code", [
    (["--kernel", "bop", "--n", "10", "--k", "2", "--p-list", "1"], 64),          # bop needs --z
    (["--kernel", "bdot", "--n", "10", "--k", "2", "--p-list", "1,x"], 64),       # bad p-list
    (["--kernel", "bdot", "--n", "10", "--k", "2", "--p-list", "0"], 64),
    (["--kernel", "bdot", "--n", "10", "--k", "4", "--p-list", "3"], 64),         # p does not divide k
    (["--kernel", "spmv", "--n", "10", "--k", "2", "--p-list", "1"], 64),
    (["--n", "10", "--k", "2", "--p-list", "1"], 64),                             # --kernel required
    (["--kernel", "bdot", "--n", "10", "--k", "2", "--p-list", "1", "--machine", "/nonexistent"], 66),
])
def test_cli_model_errors(args, code):
    assert _model(*args).returncode == code


def test_cli_model_profile_missing_key_is_unreadable(tmp_path):
    f = tmp_path / "bad.prof"
    f.write_text("peak_flops=1\nmem_bandwidth=1\n")
    assert _model("--kernel", "bdot", "--n", "1", "--k", "1", "--p-list", "1",
                  "--machine", str(f)).returncode == 66
    f.write_text("peak_flops=1\nmem_bandwidth\n")
    assert _model("--kernel", "bdot", "--n", "1", "--k", "1", "--p-list", "1",
                  "--machine", str(f)).returncode == 66
    f.write_text("peak_flops=-1\nmem_bandwidth=1\nreg_bandwidth=1\n")  # ConfigError
    assert _model("--kernel", "bdot", "--n", "1", "--k", "1", "--p-list", "1",
                  "--machine", str(f)).returncode == 64


# ------------------------------------------------------------------- theory --
@pytest.mark.parametrize("glob,p,q", [(0, 1, 1), (0, 4, 1), (0, 100, 1), (1, 4, 2), (1, 5, 3),
                                      (1, 2, 4), (1, 1, 7)])
def test_rates_match_reference(rlib, glob, p, q):
    ev = np.sort(np.random.default_rng(3).uniform(0.01, 50.0, 100))
    want = rlib.bkref_rate(glob, len(ev), _p(ev, C.c_double), p, q)
    out = run(HOST, "rate", str(glob), str(p), str(q), *["%.17g" % v for v in ev])
    assert out.returncode == 0, out.stderr
    assert float(out.stdout) == pytest.approx(want, rel=1e-15, abs=1e-16)


def test_rate_argument_errors():
    assert run(HOST, "rate", "0", "0", "1", "1.0").returncode == 2     # k = 0
    assert run(HOST, "rate", "0", "3", "1", "1", "2").returncode == 2  # k > N
    assert run(HOST, "rate", "1", "1", "0", "1").returncode == 2       # q = 0
    assert run(HOST, "rate", "0", "1", "1", "2", "1").returncode == 2  # not ascending
    assert run(HOST, "rate", "0", "1", "1", "0").returncode == 2       # not positive


@pytest.mark.parametrize("mk", MATRICES[:3])
def test_spectrum_of_matches_reference(rlib, tmp_path, mk):
    a = mk()
    f = tmp_path / "a.mtx"
    bk.save_matrix_market(str(f), a)
    out = run(HOST, "spectrum", str(f))
    assert out.returncode == 0, out.stderr
    got = np.array([float(v) for v in out.stdout.split()])
    rp, cl, vl = _csr(a)
    want = np.zeros(a.n())
    rlib.bkref_spectrum_of(a.n(), _p(rp, C.c_uint64), _p(cl, C.c_uint64), _p(vl, C.c_double),
                           _p(want, C.c_double))
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12 * want.max())
    dense = np.zeros((a.n(), a.n()))
    for r in range(a.n()):
        dense[r, cl[rp[r]:rp[r + 1]].astype(np.int64)] = vl[rp[r]:rp[r + 1]]
    np.testing.assert_allclose(got, np.linalg.eigvalsh(dense), rtol=1e-11, atol=1e-11 * want.max())


def test_spectrum_of_size_cap(tmp_path):
    f = tmp_path / "big.mtx"
    f.write_text("%%MatrixMarket matrix coordinate real symmetric\n2049 2049 2049\n" +
                 "".join(f"{i} {i} 1\n" for i in range(1, 2050)))
    assert run(HOST, "spectrum", str(f)).returncode == 2  # SizeError


# ---------------------------------------------------------------- text I/O --
@pytest.mark.parametrize("mk", MATRICES)
def test_matrix_market_writers_byte_identical(rlib, tmp_path, mk):
    a = mk()
    rp, cl, vl = _csr(a)
    ref_f, py_f, cpp_f = tmp_path / "ref.mtx", tmp_path / "py.mtx", tmp_path / "cpp.mtx"
    rlib.bkref_save_matrix_market(str(ref_f).encode(), a.n(), _p(rp, C.c_uint64),
                                  _p(cl, C.c_uint64), _p(vl, C.c_double))
    bk.save_matrix_market(str(py_f), a)
    assert run(HOST, "mm", str(ref_f), str(cpp_f)).returncode == 0
    assert py_f.read_bytes() == ref_f.read_bytes()
    assert cpp_f.read_bytes() == ref_f.read_bytes()
    b = bk.load_matrix_market(str(ref_f))
    assert b == a


MM_CASES = {
    "symmetric_comments": "%%MatrixMarket matrix coordinate real symmetric\n% a comment\n%\n"
                          "3 3 4\n1 1 4\n2 1 -1.5\n2 2 4\n3 3 2.25e-3\n",
    "general_both_triangles": "%%MatrixMarket matrix coordinate real general\n2 2 4\n"
                              "1 1 2\n1 2 0.5\n2 1 0.5\n2 2 3\n",
    "duplicates_summed": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1\n1 1 2\n2 2 5\n",
    "bad_banner": "%%MatrixMarket vector coordinate real symmetric\n1 1 1\n1 1 1\n",
    "complex": "%%MatrixMarket matrix coordinate complex symmetric\n1 1 1\n1 1 1 0\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "not_square": "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n",
    "truncated": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1\n2 2 1\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n3 1 1\n",
    "zero_index": "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n0 1 1\n",
    "no_size_line": "%%MatrixMarket matrix coordinate real symmetric\n% only comments\n",
    "empty": "",
    "general_not_symmetric": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n2 1 2\n",
}


@pytest.mark.parametrize("name", sorted(MM_CASES))
def test_matrix_market_read_semantics_match_reference(rlib, tmp_path, name):
    src = tmp_path / "in.mtx"
    src.write_text(MM_CASES[name])
    ref_o, cpp_o, py_o = tmp_path / "ref.mtx", tmp_path / "cpp.mtx", tmp_path / "py.mtx"
    rc_ref = rlib.bkref_mm_roundtrip(str(src).encode(), str(ref_o).encode())
    rc_cpp = run(HOST, "mm", str(src), str(cpp_o)).returncode
    assert rc_cpp == rc_ref
    try:
        bk.save_matrix_market(str(py_o), bk.load_matrix_market(str(src)))
        rc_py = 0
    except bk.IoError:
        rc_py = 1
    except bk.Error:
        rc_py = 2
    assert rc_py == rc_ref
    if rc_ref == 0:
        assert cpp_o.read_bytes() == ref_o.read_bytes()
        assert py_o.read_bytes() == ref_o.read_bytes()


def test_block_vector_writers_byte_identical(rlib, tmp_path):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((17, 5)) * np.logspace(-300, 300, 5)
    x[0, 0], x[1, 1], x[2, 2] = -0.0, 1.0 / 3, 5e-324
    ref_f, py_f, cpp_f = tmp_path / "ref.txt", tmp_path / "py.txt", tmp_path / "cpp.txt"
    rlib.bkref_save_block_vector(str(ref_f).encode(), 17, 5, _p(np.ascontiguousarray(x), C.c_double))
    bk.save_block_vector(str(py_f), x)
    assert run(HOST, "bv", str(ref_f), str(cpp_f)).returncode == 0
    assert py_f.read_bytes() == ref_f.read_bytes()
    assert cpp_f.read_bytes() == ref_f.read_bytes()
    y = bk.load_block_vector(str(ref_f))
    assert y.tobytes() == x.tobytes()


BV_CASES = {"ok_multiline": "2 3\n1 2\n3\n4 5 6\n", "no_header": "", "k_zero": "3 0\n",
            "early_eof": "2 2\n1 2 3\n", "junk": "2 2\n1 x 3 4\n"}


@pytest.mark.parametrize("name", sorted(BV_CASES))
def test_block_vector_read_semantics_match_reference(rlib, tmp_path, name):
    src = tmp_path / "in.txt"
    src.write_text(BV_CASES[name])
    ref_o, cpp_o = tmp_path / "ref.txt", tmp_path / "cpp.txt"
    rc_ref = rlib.bkref_bv_roundtrip(str(src).encode(), str(ref_o).encode())
    assert run(HOST, "bv", str(src), str(cpp_o)).returncode == rc_ref
    try:
        bk.load_block_vector(str(src))
        rc_py = 0
    except bk.IoError:
        rc_py = 1
    assert rc_py == rc_ref
    if rc_ref == 0:
        assert cpp_o.read_bytes() == ref_o.read_bytes()


def test_missing_files_are_io_errors(tmp_path):
    assert run(HOST, "mm", str(tmp_path / "none.mtx"), str(tmp_path / "o")).returncode == 1
    assert run(HOST, "bv", str(tmp_path / "none.txt"), str(tmp_path / "o")).returncode == 1
    with pytest.raises(bk.IoError):
        bk.load_matrix_market(str(tmp_path / "none.mtx"))


# --------------------------------------------------------- CLI (host paths) --
def test_cli_verify_rates_suite():
    out = run(CLI, "verify", "--suite", "rates")
    assert out.returncode == 0
    assert out.stdout.split() == ["rates", "convergence", "rate", "formulas", "pass"]


@pytest.mark.parametrize("args,code", [
    ([], 64), (["frobnicate"], 64), (["--help"], 0), (["solve", "--help"], 0),
    (["solve", "--nope", "1"], 64), (["solve", "--k"], 64), (["solve", "--k", "x"], 64),
    (["solve", "--k", "8", "--p", "3"], 64),                       # p must divide k
    (["solve", "--repetitions", "2", "--total-rhs", "16"], 64),    # mutually exclusive
    (["solve", "--mode", "diagonal"], 64), (["solve", "--precond", "amg"], 64),
    (["solve", "--coeff", "random"], 64), (["solve", "--repetitions", "0"], 64),
    (["solve", "--total-rhs", "12", "--k", "8"], 64),
    (["verify", "--suite", "speed"], 64),
])
def test_cli_usage_exit_codes(args, code):
    assert run(CLI, *args).returncode == code


def test_cli_rhs_file_errors(tmp_path):
    assert run(CLI, "solve", "--rhs-file", str(tmp_path / "missing.txt")).returncode == 66
    f = tmp_path / "rhs.txt"
    bk.save_block_vector(str(f), np.ones((10, 8)))  # 32x32 grid has n = 1024
    assert run(CLI, "solve", "--rhs-file", str(f)).returncode == 64
    bk.save_block_vector(str(f), np.ones((1024, 12)))  # not a multiple of k = 8
    assert run(CLI, "solve", "--rhs-file", str(f)).returncode == 64
