"""Command line mirror of the reference tool's `count` and `flagstats` commands
(proj/tools/pospopcnt.cpp:127-147, 183-215) on the GPU path.

    python -m paper_1911_02696_b200 count --input FILE|- [--kernel auto] [--k 16] [--json]
    python -m paper_1911_02696_b200 flagstats --input FILE|- [--json]

Output formats and exit codes follow the reference: 0 success, 2 usage or
input error (proj/tools/pospopcnt.cpp:43-45, 268-277).
"""
from __future__ import annotations

import argparse
import json
import sys

EXIT_OK, EXIT_MISMATCH, EXIT_USAGE = 0, 1, 2


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pospopcnt-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("count", help="positional population count of a raw little-endian word file")
    c.add_argument("--input", required=True)
    c.add_argument("--kernel", default="auto")
    c.add_argument("--k", type=int, default=16, choices=[8, 16, 32, 64])
    c.add_argument("--json", action="store_true")
    f = sub.add_parser("flagstats", help="SAM FLAG statistics of a raw little-endian u16 file")
    f.add_argument("--input", required=True)
    f.add_argument("--json", action="store_true")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK

    import numpy as np

    import paper_1911_02696_b200 as pp
    try:
        if args.cmd == "count":
            kind = pp.KernelKind.from_string(args.kernel)
            if kind is None:
                raise pp.InvalidArgument(f"unknown kernel '{args.kernel}' "
                                         "(expected scalar|csa4|csa8|csa16|forest|byteblend|auto)")
            counts, n = pp.pospopcnt_file(args.input, args.k)
            if args.json:
                print(json.dumps({"kernel": str(kind), "total_words": n, "counts": list(counts)}))
            else:
                print(f"words: {n}")
                print(f"kernel: {kind}")
                for p in range(args.k):
                    print(f"bit {p:2d}: {counts[p]}")
            return EXIT_OK
        data = sys.stdin.buffer.read() if args.input == "-" else open(args.input, "rb").read()
        if len(data) % 2:
            raise pp.InvalidArgument(f"{args.input}: odd byte length ({len(data)} bytes); "
                                     "expected raw little-endian 16-bit words")
        summary = pp.flagstats(np.frombuffer(data, np.uint16))
        if args.json:
            print(json.dumps({"pass": vars(summary.pass_), "fail": vars(summary.fail)}))
        else:
            print("field           QC-pass\tQC-fail")
            for name in ("total", "secondary", "supplementary", "n_pair_good", "n_read1", "n_read2", "n_sgltn",
                         "pair_map", "mapped", "dup"):
                print(f"{name:<16}{getattr(summary.pass_, name)}\t{getattr(summary.fail, name)}")
        return EXIT_OK
    except (pp.InvalidArgument, pp.KernelUnavailableError, pp.InvalidFlagWordError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
