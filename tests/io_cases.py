"""Loader inputs (text files) shared by the golden generator and the tests."""

from __future__ import annotations

import numpy as np


def _random_edges(seed=3, n=20000):
    rng = np.random.default_rng(seed)
    lines = ["# random edge list", ""]
    for a, b in rng.integers(0, 5000, (n, 2)).tolist():
        lines.append(f"{a}\t{b}" if a % 3 == 0 else f"{a} {b}")
    return "\n".join(lines) + "\n"


def _random_layout(seed=4, n=5000):
    rng = np.random.default_rng(seed)
    xy = rng.normal(size=(n, 2)) * 10.0 ** rng.integers(-5, 6, (n, 2))
    ids = rng.permutation(10 * n)[:n]
    lines = ["id,x,y"] + [f"{i},{x!r},{y!r}" for i, (x, y) in zip(ids.tolist(), xy.tolist())]
    return "\n".join(lines) + "\n"


EDGELISTS = {
    "simple": "0 1\n1 2\n2 0\n",
    "comments_blanks": "# c\n\n  3   4 \n4\t5\n   \n# end\n",
    "loops_dupes": "1 1\n1 2\n2 1\n2 3\n",
    "plus_leading_zeros": "+5 007\n",
    "underscores": "1_0 2\n",
    "crlf": "0 1\r\n1 2\r\n",
    "unicode_digit": "٣ 4\n",
    "negative": "-1 2\n",
    "three_tokens": "1 2 3\n",
    "not_int": "a b\n",
    "empty": "",
    "only_comments": "# x\n\n",
    "huge_id": "123456789012345678901 1\n",
    "random_20000": _random_edges(),
}

LAYOUTS = {
    "simple": "id,x,y\n0,1.5,2\n1,-3e2,0.25\n",
    "spaces": "id , x , y\n 3 , 1.0 , 2.0 \n 1,0.1,0.2\n",
    "blank_rows": "id,x,y\n\n0,1,2\n   \n7,.5,5.\n",
    "inf": "id,x,y\n0,inf,1\n",
    "nan": "id,x,y\n0,1,nan\n",
    "overflow": "id,x,y\n0,1e309,0\n",
    "subnormal": "id,x,y\n0,1e-320,4.9e-324\n",
    "duplicate": "id,x,y\n0,1,2\n0,3,4\n",
    "bad_header": "ID,x,y\n0,1,2\n",
    "empty": "",
    "header_only": "id,x,y\n",
    "four_fields": "id,x,y\n0,1,2,3\n",
    "malformed": "id,x,y\n0,abc,1\n",
    "underscores": "id,x,y\n0,1_000.5,2\n",
    "negative_id": "id,x,y\n-5,1,2\n3,4,5\n",
    "crlf": "id,x,y\r\n0,1,2\r\n",
    "random_5000": _random_layout(),
}
