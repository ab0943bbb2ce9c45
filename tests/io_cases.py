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
    # the rest of str.splitlines() / str.isspace() / int() (round 2)
    "other_breaks": "0 1\x0b1 2\x0c2 3\x1c3 4\x1d4 5\x1e5 6\x857 8\u20288 9\u20299 10\n",
    "cr_only": "1 2\r3 4\r",
    "unicode_space": "1\u3000 2\n3\u00a04\n5\x1f6\n",
    "vt_splits_line": "1\t\x0b2\n",
    "bom": "\ufeff1 2\n",
    "underscore_double": "1__0 2\n",
    "underscore_trailing": "10_ 2\n",
    "digits_4300": "1" * 4300 + " 2\n",
    "digits_4301": "1" * 4301 + " 2\n",
    "negative_big": "-" + "9" * 30 + " 1\n",
    "fullwidth_digits": "\uff11\uff12 \uff13\n",
    "sign_only": "+ 2\n",
    "comment_after_space": "   # c\n1 2\n",
    "first_error_wins": "1 2\n3\n-1 2\n",
    "overflow_then_error": "99999999999999999999 1\n1 2 3\n",
    "invalid_utf8": b"1 2\n\xff 3\n",
    "surrogate_utf8": b"1 2\n\xed\xa0\x80 3\n",
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
    # the rest of str.splitlines() / str.isspace() / int() / float() (round 2)
    "inf_word": "id,x,y\n0,Infinity,1\n",
    "nan_signed": "id,x,y\n0,-nAn,1\n",
    "unicode_digits": "id,x,y\n\u0663,\u0661.\u0665,\uff12\n",
    "float_underscore_bad": "id,x,y\n0,1_.5,2\n",
    "float_exp_underscore": "id,x,y\n0,1e1_0,2\n",
    "line_separators": "id,x,y\u20280,1,2\u20291,3,4\n",
    "header_unicode_spaces": "\u3000id ,\tx, y\u00a0\n0,1,2\n",
    "bom_header": "\ufeffid,x,y\n0,1,2\n",
    "dup_before_malformed": "id,x,y\n1,0,0\n1,2,2\n3,a,b\n",
    "malformed_before_dup": "id,x,y\n1,0,0\n2,a,b\n1,2,2\n",
    "dup_three": "id,x,y\n5,0,0\n6,0,0\n5,1,1\n6,1,1\n5,2,2\n",
    "nonfinite_and_dup": "id,x,y\n1,0,0\n1,inf,0\n",
    "int_id_float": "id,x,y\n1.0,2,3\n",
    "hex_float": "id,x,y\n0,0x1p3,2\n",
    "big_id": "id,x,y\n123456789012345678901,1,2\n",
    "empty_field": "id,x,y\n0,,1\n",
    "only_blank_rows": "id,x,y\n  \n\t\n",
    "header_crlf": "id,x,y\r\n",
    "quote_in_row": "id,x,y\n0,'1\",2,3\n",
    "invalid_utf8": b"id,x,y\n0,1,\xff\n",
}
