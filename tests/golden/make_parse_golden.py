"""Regenerate tests/golden/parse_golden.json from the REFERENCE's own text
ingestion (pkg/src/bflybfs/graphs.py load_edge_list / write_edge_list,
graphs.py:96-209), imported from /root/reference.

Each case is raw input bytes (base64) plus what the reference returns for it
read from a path: the edges (hash + first pairs) and num_vertices, or the
ParseError line number and message.  Run in the build container:
    python tests/golden/make_parse_golden.py
"""

from __future__ import annotations

import base64
import hashlib
import io
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

H = b"%%MatrixMarket matrix coordinate pattern general\n"

CASES = [
    # ---- "edges" format (graphs.py:109-134)
    ("edges", "basic", b"0 1\n1 2\n2 0\n"),
    ("edges", "comments_blank", b"# comment\n\n% other\n   3  4  \n\t\n5 6\n"),
    ("edges", "crlf", b"0 1\r\n2 3\r\n"),
    ("edges", "lone_cr", b"0 1\r2 3\r4 5"),
    ("edges", "no_final_newline", b"0 1\n5 6"),
    ("edges", "odd_whitespace", b"0\t1\n\x0b2 3\x0c\n7\x1c8\n"),
    ("edges", "signs_underscores", b"+1 1_0\n-0 3\n0007 2_2_2\n"),
    ("edges", "max_vid", b"4294967295 0\n"),
    ("edges", "empty", b""),
    ("edges", "only_comments", b"# a\n% b\n\n"),
    ("edges", "indented_comment", b"   # c d e\n1 2\n"),
    ("edges", "self_loops_dups", b"1 1\n1 2\n1 2\n2 1\n"),
    ("edges", "err_three_tokens", b"0 1\n1 2 3\n4 5\n"),
    ("edges", "err_one_token", b"0 1\n7\n"),
    ("edges", "err_nonint", b"0 1\nx 2\n"),
    ("edges", "err_float", b"1.5 2\n"),
    ("edges", "err_double_underscore", b"1__0 2\n"),
    ("edges", "err_leading_underscore", b"_1 2\n"),
    ("edges", "err_trailing_underscore", b"1_ 2\n"),
    ("edges", "err_hex", b"0x10 1\n"),
    ("edges", "err_sign_only", b"+ 1\n"),
    ("edges", "err_negative", b"0 1\n-1 2\n"),
    ("edges", "err_negative_dst", b"3 -7\n"),
    ("edges", "err_range_src", b"0 1\n4294967296 1\n"),
    ("edges", "err_range_dst", b"1 4294967296\n"),
    ("edges", "err_range_huge", b"99999999999999999999999 1\n"),
    ("edges", "err_first_wins", b"0 1\n\na b c\nx y\n-1 -1\n"),
    ("edges", "err_non_ascii", b"0 1\n\xc3\xa9 2\n"),
    ("edges", "err_nonint_before_negative", b"-1 x\n"),
    # ---- "mtx" format (graphs.py:137-182)
    ("mtx", "basic", H + b"% comment\n3 3 2\n1 2\n3 1\n"),
    ("mtx", "values_ignored", b"%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 0.5\n2 1 7 extra\n"),
    ("mtx", "rect", H + b"2 5 1\n2 5\n"),
    ("mtx", "crlf", b"%%MatrixMarket Matrix Coordinate pattern symmetric\r\n3 3 1\r\n2 3\r\n"),
    ("mtx", "zero", H + b"0 0 0\n"),
    ("mtx", "blank_lines", H + b"\n\n2 2 1\n\n1 1\n\n"),
    ("mtx", "err_no_header", b""),
    ("mtx", "err_array_header", b"%%MatrixMarket matrix array real general\n2 2\n1\n"),
    ("mtx", "err_garbage_header", b"hello\n1 1 0\n"),
    ("mtx", "err_size_tokens", H + b"3 3\n"),
    ("mtx", "err_size_nonint", H + b"3 x 2\n"),
    ("mtx", "err_missing_size", H + b"% only comments\n"),
    ("mtx", "err_entry_tokens", H + b"3 3 1\n1\n"),
    ("mtx", "err_entry_nonint", H + b"3 3 1\n1 a\n"),
    ("mtx", "err_outside", H + b"3 3 1\n4 1\n"),
    ("mtx", "err_zero_index", H + b"3 3 1\n0 1\n"),
    ("mtx", "err_negative_index", H + b"3 3 1\n-1 2\n"),
    ("mtx", "err_hash_line", H + b"3 3 1\n# c\n"),
    ("mtx", "err_count_short", H + b"3 3 2\n1 2\n"),
    ("mtx", "err_count_long", H + b"3 3 1\n1 2\n2 3\n"),
]


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    sys.path.insert(0, REF_SRC)
    from bflybfs import graphs

    out = {"_provenance": "reference /root/reference/pkg/src/bflybfs/graphs.py load_edge_list "
                          "(path source) and write_edge_list; tests/golden/make_parse_golden.py",
           "cases": []}
    with tempfile.TemporaryDirectory() as tmp:
        for fmt, name, data in CASES:
            path = os.path.join(tmp, name)
            with open(path, "wb") as fh:
                fh.write(data)
            rec = {"fmt": fmt, "name": name, "data_b64": base64.b64encode(data).decode()}
            try:
                el = graphs.load_edge_list(path, fmt)
                rec.update(num_vertices=int(el.num_vertices), num_edges=int(el.num_edges),
                           edges_sha=sha16(el.edges), edges_head=el.edges[:8].tolist())
                # write_edge_list output bytes
                wpath = os.path.join(tmp, name + ".out")
                graphs.write_edge_list(el, wpath)
                with open(wpath, "rb") as fh:
                    rec["written_sha"] = hashlib.sha256(fh.read()).hexdigest()[:16]
            except graphs.ParseError as e:
                rec.update(error=str(e), line_no=e.line_no)
            # the same bytes as a text stream (io.StringIO splits on "\n" only)
            if all(b < 128 for b in data):
                try:
                    el2 = graphs.load_edge_list(io.StringIO(data.decode("ascii")), fmt)
                    rec["stream"] = {"num_vertices": int(el2.num_vertices),
                                     "edges_sha": sha16(el2.edges)}
                except graphs.ParseError as e:
                    rec["stream"] = {"error": str(e)}
            out["cases"].append(rec)
    with open(os.path.join(HERE, "parse_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"{len(out['cases'])} cases")


if __name__ == "__main__":
    main()
