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
