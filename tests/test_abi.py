"""CPU tests of the drop-in boundary (no GPU needed).

* libqfb.so loads and exports every entry point include/qfb.h declares;
* host-side entry points (config, scale math, validation) are bit-identical
  to the reference's and raise the reference's error taxonomy;
* device entry points validate before touching the GPU;
* the C++ mirror include/qfb.hpp compiles against the reference's own
  qf::Tensor / qf::QuantConfig types (drop-in by template) and runs its
  host-only parts.
"""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "qfb.h")
LIB = os.path.join(ROOT, "paper_2511_12653_b200", "libqfb.so")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qfb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (qfb_\w+)", out))
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for n in names:
        assert getattr(lib, n) is not None


def test_no_oracle_or_torch_dependency():
    """The product library links neither the oracle nor torch."""
    out = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "orc" not in out and "qfref" not in out and "torch" not in out
    dyn = subprocess.run(["nm", "-D", LIB], capture_output=True, text=True).stdout
    assert "orc_" not in dyn and "ref_" not in dyn.replace("pref_", "")


def test_host_scale_math_matches_reference(qfb, ref):
    rng = np.random.default_rng(0)
    for x in np.concatenate([rng.uniform(-45, 45, 3000), [0.0, 30.0, -30.0, 30.5]]):
        assert qfb.softplus(x) == ref.softplus(x)
        assert qfb.sigmoid(x) == ref.sigmoid(x)
        assert qfb.resolve_scale(x) == ref.resolve_scale(x)[1]
        assert qfb.resolve_scale(x, None, qfb.PREC_HALF) == ref.resolve_scale(x, 1)[1]
    for y in rng.uniform(1e-6, 40, 500):
        assert qfb.softplus_inv(y) == ref.softplus_inv(y)[1]


def test_scale_grad_factors_match_reference_chain(qfb, ref):
    # chain = clamped ? 0 : sigmoid (quant.hpp:242-244)
    ls = [-100.0, -14.0, -5.0, 0.0, 3.0, 70.0]
    s, ch = qfb.scale_grad_factors(ls)
    assert s == [ref.resolve_scale(v)[1] for v in ls]
    assert ch[0] == 0.0 and ch[-1] == 0.0      # clamped at s_min / s_max
    assert ch[2] == ref.sigmoid(-5.0)


def test_error_taxonomy_host_side(qfb):
    with pytest.raises(qfb.NonFiniteError):
        qfb.resolve_scale(float("nan"))
    with pytest.raises(qfb.ValueError):
        qfb.softplus_inv(0.0)
    with pytest.raises(qfb.ValueError):
        qfb.cast_scales_f32([0.5, 0.0])
    with pytest.raises(qfb.ValueError):
        qfb.QuantConfig(eps=1e-3).validate()     # test_quant.cpp:38-43
    with pytest.raises(qfb.ValueError):
        qfb.QuantConfig(bits=1).validate()
    assert qfb.QuantConfig().q_max() == 127
    assert qfb.cast_scales_f32([0.1]) == [np.float32(0.1)]


def test_device_entry_points_validate_first(qfb):
    L = qfb.lib()
    assert L.qfb_fq_fwd(None, 0, None, None, 1, 1, 1, None, 127, 0) == 2
    assert b"null qfb_ctx" in L.qfb_last_error()
    assert L.qfb_fq_bwd(None, 0, None, None, None, 1, 1, 1, None, None, 127, None, 0) == 2
    assert L.qfb_status_name(1) == b"ShapeError"
    assert L.qfb_status_name(6) == b"FusedPathError"


def test_ctx_create_without_gpu_is_a_cuda_error(qfb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = qfb.lib().qfb_ctx_create(0, None, ctypes.byref(h))
    assert st in (2, 7)   # no device -> ValueError(range) or CudaError


def test_cpp_mirror_compiles_against_reference_types(tmp_path):
    """qfb.hpp is a template drop-in for qf::Tensor (compile + host-only run)."""
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers absent (GPU box)")
    src = tmp_path / "dropin.cpp"
    src.write_text(r'''
#include <cstdio>
#include <span>
#include "quantfuse/distill.hpp"
#include "quantfuse/quant.hpp"
#include "quantfuse/tensor_io.hpp"
#include "qfb.hpp"
int main() {
  qf::QuantConfig cfg;
  // formats (host only): our writers/readers round-trip the reference's
  {
    qf::Tensor t({2, 3}, {1, -2, 3, 4.5f, -0.0f, 6}, qf::Precision::EmulatedHalf);
    qf::save_tensor("t_ref.qsim", t);
    qf::Tensor u = qfb::load_tensor<qf::Tensor>("t_ref.qsim");
    if (u.shape != t.shape || u.data != t.data || u.precision != t.precision) return 4;
    qfb::save_tensor("t_qfb.qsim", u);
    if (qf::read_file("t_qfb.qsim") != qf::read_file("t_ref.qsim")) return 5;
    qf::ScaleSet set;
    set.by_layer["conv1"] = qf::ScaleParams{{-3.0, -2.5}, -1.25};
    set.by_layer["fnet_out"] = qf::ScaleParams{{-4.0}, -2.0};
    qf::save_scales("s_ref.qscl", set);
    qfb::ScaleMap m = qfb::load_scales("s_ref.qscl");
    if (m.size() != 2 || m["conv1"].first.size() != 2 || m["fnet_out"].second != -2.0) return 6;
    qfb::save_scales("s_qfb.qscl", set);
    if (qf::read_file("s_qfb.qscl") != qf::read_file("s_ref.qscl")) return 7;
  }
  // host scale math: bit-identical to the reference
  for (double ls : {-30.0, -3.0, 0.0, 2.5}) {
    if (qfb::resolve_scale(ls, cfg) != qf::resolve_scale(ls, cfg)) return 1;
  }
  try {
    qfb::Context ctx(0);           // no GPU in the build container
    qf::Tensor x({2, 3}, {1, 2, 3, 4, 5, 6});
    std::vector<double> s = {0.1, 0.2};
    qf::Tensor y = qfb::fake_quantize(ctx, x, std::span<const double>(s), cfg);
    qf::Tensor y_ref = qf::fake_quantize(x, std::span<const double>(s), cfg);
    auto g = qfb::fake_quantize_backward(ctx, x, std::span<const double>(s), cfg, x, qf::Precision::Full);
    auto dl = qfb::distill_loss(ctx, x, x, x, x, 1.0);
    return y.data == y_ref.data && g.d_log_scale.size() == 2 && dl.total == 0.0 ? 0 : 3;
  } catch (const qfb::CudaError&) {
    std::puts("no-gpu");
    return 0;
  } catch (const qfb::ValueError&) {
    std::puts("no-gpu");
    return 0;
  }
}
''')
    exe = tmp_path / "dropin"
    json_inc = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ref_inc}", f"-I{json_inc}", f"-I{ROOT}/include", str(src),
                    "-o", str(exe), LIB, f"-Wl,-rpath,{os.path.dirname(LIB)}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, cwd=str(tmp_path))
    assert r.returncode == 0, r.stdout + r.stderr


def test_nccl_loads_at_run_time():
    """libqfb has no link-time NCCL dependency (dlopen at the call); in this
    image the system libnccl.so.2 is found, so the exchange is available."""
    import subprocess
    from paper_2511_12653_b200 import LIB_PATH, nccl_available
    deps = subprocess.run(["readelf", "-d", LIB_PATH], capture_output=True, text=True).stdout
    assert "nccl" not in deps.lower()
    assert nccl_available()


def test_plain_c_client(tmp_path):
    """include/qfb.h is a C header: a C11 program compiled with gcc links
    against libqfb.so and calls the host entry points (scale math, error
    taxonomy, QSIM serialization) — the binding an FFI (cgo, ctypes, JNI
    shim) would generate. No GPU needed."""
    import subprocess
    from paper_2511_12653_b200 import LIB_PATH
    src = tmp_path / "client.c"
    src.write_text(r'''
#include <stdio.h>
#include <string.h>
#include "qfb.h"
int main(void) {
  qfb_quant_config cfg;
  qfb_quant_config_default(&cfg);
  if (qfb_quant_config_validate(&cfg) != QFB_OK || qfb_q_max(&cfg) != 127) return 1;
  double ls[3] = {-4.0, 0.0, 2.0}, s[3];
  if (qfb_resolve_scales(ls, 3, &cfg, QFB_PREC_FULL, s) != QFB_OK) return 2;
  if (!(s[0] > 0.0 && s[1] > s[0] && s[2] > s[1])) return 3;
  double bad = 0.0 / 0.0;
  if (qfb_resolve_scales(&bad, 1, &cfg, QFB_PREC_FULL, s) != QFB_ERR_NONFINITE) return 4;
  if (strlen(qfb_last_error()) == 0) return 5;
  float data[6] = {1, 2, 3, 4, 5, 6};
  int64_t shape[2] = {2, 3};
  size_t n = 0;
  if (qfb_qsim_serialize(data, 2, shape, 0, NULL, 0, &n) != QFB_OK || n != 13 + 16 + 24) return 6;
  printf("ok %s\n", qfb_build_info());
  return 0;
}
''')
    exe = tmp_path / "client"
    libdir = os.path.dirname(LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-O1", f"-I{ROOT}/include", str(src), "-o", str(exe),
                    f"-L{libdir}", "-lqfb", f"-Wl,-rpath,{libdir}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert r.stdout.startswith("ok ")


def test_reference_arm_maps_no_product_library():
    """bench.py --impl reference times the reference's own code only: the
    process maps oracle/_ref/libqfref.so and NOT libqfb.so (the package's
    binding loads lazily; the arm imports only the pure-Python shapes), and
    its `config` is the GPU arm's (the same bench_config function)."""
    import json
    import oracle
    if not oracle.reference_available():
        pytest.skip("reference build absent")
    code = r"""
import io, json, sys, contextlib, runpy
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0", "--no-single-thread"]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    try:
        runpy.run_path("bench.py", run_name="__main__")
    except SystemExit:
        pass
maps = open("/proc/self/maps").read()
line = [l for l in buf.getvalue().splitlines() if l.startswith("{")][-1]
print(json.dumps({"line": json.loads(line), "qfb": "libqfb.so" in maps, "ref": "libqfref.so" in maps}))
"""
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["ref"] and not d["qfb"]
    assert d["line"]["impl"] == "reference"
    sys.path.insert(0, ROOT)
    import bench
    args = bench.parse_args_list(["--steps", "1", "--warmup", "0"])
    assert d["line"]["config"] == bench.bench_config(args, 1)
    assert d["line"]["data"] == bench.DATA
