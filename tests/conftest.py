"""Shared fixtures.  `-m gpu` tests need a CUDA device (run on the B200 box);
everything else runs on CPU.  The native libraries are built on demand."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    lib = os.path.join(ROOT, "paper_1011_5599_b200", "libhanf.so")
    port = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-j8", "-C", os.path.join(ROOT, "paper_1011_5599_b200", "csrc")],
                       check=True)
    if not os.path.exists(port):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)


@pytest.fixture(scope="session")
def hanf():
    import paper_1011_5599_b200 as m
    return m


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.have_ref():
        pytest.skip("reference engine (oracle/_ref) not built here")
    return oracle.ref()


@pytest.fixture(scope="session")
def traces():
    with open(os.path.join(GOLDEN, "engine_traces.json")) as f:
        return json.load(f)["cases"]


@pytest.fixture(scope="session")
def primitives():
    with open(os.path.join(GOLDEN, "primitives.json")) as f:
        return json.load(f)["layouts"]


@pytest.fixture(scope="session")
def recorded():
    with open(os.path.join(GOLDEN, "recorded.json")) as f:
        return json.load(f)


def graph_of(hanf, spec):
    """Rebuilds a golden case's graph with the product's generators."""
    kind = spec["kind"]
    if kind == "uniform_random":
        return hanf.gen_uniform_random(spec["n"], spec["d"], spec["seed"])
    if kind == "clique_path":
        return hanf.gen_clique_path(spec["k"], spec["l"])
    if kind == "edges":
        return hanf.Graph.from_edges(spec["n"], spec["edges"])
    if kind == "path":
        return hanf.Graph.from_edges(spec["n"], [(v, v + 1) for v in range(spec["n"] - 1)])
    if kind == "rmat":
        return hanf.gen_rmat(spec["scale"], spec["edge_factor"], 0.57, 0.19, 0.19, spec["seed"],
                             spec["permute_seed"])
    raise ValueError(kind)
