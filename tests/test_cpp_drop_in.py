"""GPU: the C++ drop-in header (include/demb200/simulation.hpp) driven side by side with the
reference demforge::Simulation in one C++ program (tests/cpp/drop_in_test.cpp)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "drop_in_test")


@pytest.mark.gpu
def test_cpp_drop_in_side_by_side(cuda):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/drop_in_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout


@pytest.mark.gpu
def test_cpp_namespace_alias_switch(cuda):
    """tests/cpp/alias_test.cpp: a reference-API program compiled with `namespace demforge =
    demb200;` — every member and free function of pipeline.hpp:50-107 with the reference's types."""
    binp = os.path.join(HERE, "cpp", "alias_test")
    if not os.path.exists(binp):
        pytest.skip("tests/cpp/alias_test not built")
    r = subprocess.run([binp], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "PASSED" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_sharded_simulation(cuda):
    """tests/cpp/shard_test.cpp: the C++ multi-GPU entry point (include/demb200/sharded.hpp over
    dem_create_sharded / dem_shard_*) for 1-4 ranks, walled and periodic Lees-Edwards, bitwise
    against one demb200::Simulation — no Python in the loop."""
    binp = os.path.join(HERE, "cpp", "shard_test")
    if not os.path.exists(binp):
        pytest.skip("tests/cpp/shard_test not built")
    r = subprocess.run([binp], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "PASSED" in r.stdout, r.stdout + r.stderr
