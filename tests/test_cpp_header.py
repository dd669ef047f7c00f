"""The reference's Catch2 cases restated in C++ against include/cvgram/*.hpp
(tests/cpp/test_header_api.cpp), i.e. the drop-in boundary for C++ callers."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_header_api")


def _run(*args):
    r = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    return r


def test_cpp_header_host_cases():
    assert os.path.exists(BIN), "built by __graft_entry__.build()"
    r = _run("--host")
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_header_all_cases_on_device():
    r = _run()
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failing tests" in r.stdout


@pytest.mark.gpu
def test_cpp_header_all_cases_on_a_multi_device_context():
    """The same C++ cases with CVG_DEVICES naming a repeated device: every cvgram::run_all_folds call goes
    through cvg_context_create_multi's sharded path (rank plans on host threads, device-copy exchanges)."""
    env = dict(os.environ, CVG_DEVICES="0,0")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failing tests" in r.stdout


def test_headers_compile_against_eigen_typedefs():
    """With <Eigen/Dense> on the include path the headers take the reference's own Matrix / Vector / Index
    typedefs (core.hpp:16-18), so callers' Eigen code on a FoldResult compiles unchanged.  Eigen is absent from
    this image: tests/cpp/eigen_shape stands in with Eigen's spelling of the members the headers may use."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-I" + os.path.join(root, "include"),
                        "-I" + os.path.join(root, "tests", "cpp", "eigen_shape"),
                        os.path.join(root, "tests", "cpp", "eigen_shape_check.cpp")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
