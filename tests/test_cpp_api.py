"""The C++ drop-in API (reference names, namespace reshard) used directly from C++:
examples/plan_cli.cpp compiles against paper_2312_05181_b200/csrc headers, links
libreshard_b200.so and reproduces the Fig. 6 golden plan (acceptance #4) and the SPEC.md:268
text format; error codes surface as process exit 1 + Errc."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2312_05181_b200")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


@pytest.fixture(scope="module")
def plan_cli(rs, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "plan_cli")
    subprocess.run([CXX, "-std=c++20", "-O1", "-I", os.path.join(PKG, "csrc"), os.path.join(ROOT, "examples", "plan_cli.cpp"),
                    "-L", PKG, "-lreshard_b200", f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


def test_fig6_from_cpp(plan_cli):
    p = subprocess.run([plan_cli, "fig6"], capture_output=True, text=True, check=True)
    golden = open(os.path.join(ROOT, "tests", "golden", "fig6_plan.txt")).read()
    plan = "".join(line + "\n" for line in p.stdout.splitlines() if not line.startswith("#"))
    assert plan == golden
    assert "# total=36" in p.stdout


def test_cpp_plan_equals_c_abi_plan(plan_cli, rs):
    p = subprocess.run([plan_cli, "gpt", "4", "2", "1", "2", "2", "2"], capture_output=True, text=True, check=True)
    cat = rs.Catalog.gpt(64, 4, 16, 128, rs.MIXED_ADAM)
    a = cat.build_strategy([(0, i) for i in range(8)], 4, 2, 1)
    b = cat.build_strategy([(0, i) for i in range(8)], 2, 2, 2)
    text = rs.generate_plan(a, b).text()
    assert "".join(line + "\n" for line in p.stdout.splitlines() if not line.startswith("#")) == text


def test_cpp_error_code(plan_cli):
    p = subprocess.run([plan_cli, "gpt", "3", "1", "1", "1", "1", "1"], capture_output=True, text=True)
    assert p.returncode == 1 + 9 and p.stderr.startswith("IndivisibleSliceDim")  # 64 % 3 != 0


def test_planner_clean_under_asan_ubsan(plan_cli, tmp_path):
    """The host planner (core / ptc / planner sources, no CUDA) built with AddressSanitizer
    and UndefinedBehaviorSanitizer: the Fig. 6 plan, the BASELINE 6.7B transitions and an
    error path run without a sanitizer report and print exactly what the normal build
    prints (host ASan/UBSan)."""
    asan = str(tmp_path / "plan_cli_asan")
    host = os.path.join(PKG, "csrc", "host")
    subprocess.run([CXX, "-std=c++20", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
                    "-fno-omit-frame-pointer", "-I", os.path.join(PKG, "csrc"),
                    os.path.join(ROOT, "examples", "plan_cli.cpp"),
                    *[os.path.join(host, f) for f in ("core.cpp", "ptc.cpp", "planner.cpp")], "-o", asan], check=True)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0", UBSAN_OPTIONS="print_stacktrace=1")
    for args in (["fig6"], ["gpt", "4", "2", "1", "2", "2", "2", "4096", "32", "2048", "50304"],
                 ["gpt", "2", "2", "2", "2", "2", "1"], ["gpt", "2", "1", "1", "1", "2", "1", "768", "12", "1024", "50304"],
                 ["gpt", "3", "1", "1", "1", "1", "1"]):
        want = subprocess.run([plan_cli, *args], capture_output=True, text=True)
        got = subprocess.run([asan, *args], capture_output=True, text=True, env=env)
        assert "Sanitizer" not in got.stderr and "runtime error" not in got.stderr, got.stderr[-2000:]
        assert (got.returncode, got.stdout) == (want.returncode, want.stdout)


@pytest.fixture(scope="module")
def tensor_values(rs, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "tensor_values")
    subprocess.run([CXX, "-std=c++20", "-O1", "-I", os.path.join(PKG, "csrc"),
                    os.path.join(ROOT, "examples", "tensor_values.cpp"), "-L", PKG, "-lreshard_b200",
                    f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


EXPECTED_ERRORS = ["zero extent: InvalidTensor", "payload size: InvalidTensor", "slice out of bounds: RangeOutOfBounds",
                   "merge gap: TilingGap", "merge overlap: TilingOverlap"]


def test_reference_tensor_value_api_validation(tensor_values, rs):
    """reshard::Tensor / slice / merge with the reference's signatures (tensor.hpp:16-47):
    construction and argument errors come out with the reference's Errc before any device
    work; without a GPU the first data operation fails with DeviceUnavailable."""
    p = subprocess.run([tensor_values], capture_output=True, text=True)
    assert p.stdout.splitlines()[:5] == EXPECTED_ERRORS
    import struct

    iota = b"".join(struct.pack("<f", float(i)) for i in range(24))
    assert p.stdout.splitlines()[5] == "refine:[0:2][2:3][3:4][4:6] splitmix64(0) e220a8397b1dcdaf dtype f32"
    assert p.stdout.splitlines()[6] == f"digest {rs.fnv1a64(iota):016x}"  # reshard::fnv1a64(std::span)
    assert p.stdout.splitlines()[7] == "ptx round trip: equal (118 bytes, encoded_size 118)"  # 4+1+1+2*8 + 96
    if rs.device_count() == 0:
        assert p.returncode == 1 + rs._capi.ERRC.index("DeviceUnavailable")
        assert p.stderr.startswith("DeviceUnavailable")


@pytest.mark.gpu
def test_reference_tensor_value_api_on_gpu(tensor_values):
    """The same program on a B200: SPEC.md:60-62's slice and the quadrant round trip."""
    p = subprocess.run([tensor_values], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    lines = p.stdout.splitlines()
    assert lines[:5] == EXPECTED_ERRORS
    assert lines[8] == "slice [0:4,2:4]: 2 3 8 9 14 15 20 21"
    assert lines[9] == "quadrant round trip: equal"


@pytest.fixture(scope="module")
def reshard_cli(rs, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "reshard_cli")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run([CXX, "-std=c++20", "-O1", "-I", os.path.join(PKG, "csrc"), "-I", os.path.join(cuda, "include"),
                    os.path.join(ROOT, "examples", "reshard_cli.cpp"), "-L", PKG, "-lreshard_b200",
                    "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


def test_reshard_cli_compiles_and_fails_loudly_without_gpu(reshard_cli, rs):
    """The whole reconfiguration driven from C++ (examples/reshard_cli.cpp): without a GPU
    it stops with DeviceUnavailable (no CPU path)."""
    if rs.device_count() > 0:
        pytest.skip("a GPU is visible")
    p = subprocess.run([reshard_cli], capture_output=True, text=True)
    assert p.returncode == 1 + rs._capi.ERRC.index("DeviceUnavailable") and p.stderr.startswith("DeviceUnavailable")


@pytest.mark.gpu
def test_reshard_cli_on_gpu(reshard_cli):
    """examples/reshard_cli.cpp on a B200: GPT-2 small (2,1,1) -> (1,2,1) and GPT-3 1.3B
    (2,1,1) -> (2,1,2) from C++, every destination byte verified."""
    for args in (["768", "12", "1024", "50304", "2", "1", "1", "1", "2", "1"], []):
        p = subprocess.run([reshard_cli, *args], capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr
        assert "mismatched bytes 0" in p.stdout


def test_c_abi_header_is_plain_c(rs, tmp_path):
    """include/reshard_b200.h is the drop-in boundary for cgo / JNI / N-API / ctypes: it must
    compile as ISO C11 (-pedantic, no C++), and a C program links libreshard_b200.so and
    calls through it (no GPU needed for the error table)."""
    src = tmp_path / "abi.c"
    src.write_text('#include "reshard_b200.h"\n#include <string.h>\n'
                   'int main(void) {\n'
                   '  rs_range r;\n'
                   '  if (rs_range_parse("[0:3,2:4]", &r) != 0 || r.rank != 2 || r.hi[1] != 4) return 2;\n'
                   '  if (rs_range_parse("[x:1]", &r) == 0) return 3;\n'
                   '  if (strchr(rs_last_error(), \':\') == NULL) return 4;  /* "<ErrcName>: <detail>" */\n'
                   '  return rs_errc_count() > 0 ? 0 : 5;\n}\n')
    out = str(tmp_path / "abi")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"),
                    str(src), "-L", PKG, "-lreshard_b200", f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    assert subprocess.run([out]).returncode == 0


@pytest.fixture(scope="module")
def dataset_cli(rs, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "dataset_cli")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run([CXX, "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(PKG, "csrc"), "-I",
                    os.path.join(cuda, "include"), os.path.join(ROOT, "examples", "dataset_cli.cpp"), "-L", PKG,
                    "-lreshard_b200", "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{PKG}", "-o", out],
                   check=True)
    return out


def test_dataset_cli_validates_then_fails_loudly_without_gpu(dataset_cli, rs):
    """examples/dataset_cli.cpp (the dataset module from C++): SPEC errors come before any
    device work; without a GPU it stops with DeviceUnavailable (no CPU path)."""
    p = subprocess.run([dataset_cli, "1000", "48", "0", "5", "7"], capture_output=True, text=True)
    assert p.returncode == 1 + rs._capi.ERRC.index("IndivisibleBatch") and p.stderr.startswith("IndivisibleBatch")
    if rs.device_count() > 0:
        return
    p = subprocess.run([dataset_cli], capture_output=True, text=True)
    assert p.returncode == 1 + rs._capi.ERRC.index("DeviceUnavailable") and p.stderr.startswith("DeviceUnavailable")


@pytest.mark.gpu
def test_dataset_cli_on_gpu(dataset_cli):
    """examples/dataset_cli.cpp on a B200: the GPU shuffle equals the host loop and a fused batch
    of every new rank matches the closed-form positions, the index and the offsets."""
    for args in ([], ["100003", "64", "700", "8", "13"], ["5000", "40", "124", "4", "3"]):
        p = subprocess.run([dataset_cli, *args], capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stdout + p.stderr
        assert "identical to the host loop" in p.stdout and "mismatches 0" in p.stdout
