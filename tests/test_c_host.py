"""The C ABI from a non-Python host (tests/c_host/glare_host.c): the header
compiles as C11 and links against libglare_b200.so with gcc (CPU), and on a
B200 the C program's five metrics, its `world`-way interleaved shards and
its NCCL combine through the library equal the oracle (counts exact, reals
1e-9 relative)."""

from __future__ import annotations

import json
import math
import os
import shutil
import struct
import subprocess

import numpy as np
import pytest

import cases
from conftest import REPO, graph_from, strict_close

SRC = os.path.join(REPO, "tests", "c_host", "glare_host.c")
LIBDIR = os.path.join(REPO, "paper_2411_09809_b200", "_lib")
CUDA = "/usr/local/cuda"


def _build(tmp_path) -> str:
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "glare_host")
    cmd = ["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-O2",
           "-I", os.path.join(REPO, "include"), "-I", os.path.join(CUDA, "include"),
           SRC, "-o", exe, "-L", LIBDIR, "-lglare_b200", "-L", os.path.join(CUDA, "lib64"),
           "-lcudart", f"-Wl,-rpath,{LIBDIR}:{os.path.join(CUDA, 'lib64')}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_host_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


def _write(path, g, r, ideal):
    with open(path, "wb") as f:
        f.write(struct.pack("<qqdd", g.num_vertices, g.num_edges, r, ideal))
        f.write(np.ascontiguousarray(g.xy, dtype=np.float64).tobytes())
        f.write(np.ascontiguousarray(g.edges, dtype=np.int64).tobytes())


@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("lattice", 3), ("c1", 8), ("near_collinear", 2)])
def test_c_host_matches_oracle(gpu, tmp_path, name, world):
    from oracle import glare_oracle as O
    from oracle import sweep as S
    from paper_2411_09809_b200 import configs

    if name == "c1":
        g, p = configs.config1()
        r = p["radius"]
    else:
        g = graph_from(cases.lattice_stress if name == "lattice" else cases.near_collinear)
        r = 1.0 if name == "lattice" else 0.01
    ideal = 7.0 * math.pi / 18.0
    exe = _build(tmp_path)
    inp = tmp_path / "in.bin"
    _write(inp, g, r, ideal)
    out = subprocess.run([exe, str(inp), str(world)], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    c, d = S.crossing_scan(g.xy, g.edges, ideal)
    assert int(res["ec"]) == c and strict_close(res["dev"], d)
    assert int(res["ec_sharded"]) == c and strict_close(res["dev_sharded"], d)
    assert int(res["nc"]) == S.node_occlusion(g.xy, r)
    assert strict_close(res["ma"], O.minimum_angle(g.xy, g.edges))
    assert strict_close(res["ml"], O.edge_length_variation(g.xy, g.edges))
    assert res["chunk"] == O.interleaved_chunk(-(-g.num_edges // 256) * (-(-g.num_edges // 256) + 1) // 2, world)
