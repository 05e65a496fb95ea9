"""Command line mirror of the reference tool's `count` and `flagstats` commands
(proj/tools/pospopcnt.cpp:127-147, 183-215) on the GPU path.

    python -m paper_1911_02696_b200 count --input FILE|- [--kernel auto] [--k 16] [--json]
    python -m paper_1911_02696_b200 flagstats --input FILE|- [--mode reference|pospopcnt|differential] [--json]

Output formats and exit codes follow the reference: 0 success, 2 usage or
input error (proj/tools/pospopcnt.cpp:43-45, 268-277).
"""
from __future__ import annotations

import argparse
import json
import sys

EXIT_OK, EXIT_MISMATCH, EXIT_USAGE = 0, 1, 2


def _format(summary) -> str:
    """format_flag_summary (proj/core/src/flagstats.cpp:147-164)."""
    lines = ["field           QC-pass\tQC-fail"]
    for name in ("total", "secondary", "supplementary", "n_pair_good", "n_read1", "n_read2", "n_sgltn",
                 "pair_map", "mapped", "dup"):
        lines.append(f"{name:<16}{getattr(summary.pass_, name)}\t{getattr(summary.fail, name)}")
    return "\n".join(lines) + "\n"


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
    f.add_argument("--mode", default="pospopcnt",
                   help="reference|pospopcnt|differential (reference tool option; both summaries come from the GPU: "
                        "differential cross-checks the byte-frame FLAG kernel against the 16-bit-lane one)")
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
        if args.mode not in ("reference", "pospopcnt", "differential"):
            raise pp.InvalidArgument(f"unknown mode '{args.mode}' (expected reference|pospopcnt|differential)")
        words = np.frombuffer(data, np.uint16)
        summary = pp.flagstats(words)
        if args.mode == "differential":  # pospopcnt.cpp:194-209, two GPU kernels instead of two CPU paths
            import os
            prev = os.environ.get("POSPOP_FLAG_VARIANT")
            os.environ["POSPOP_FLAG_VARIANT"] = "6,32,0,512,2"  # the 16-bit-lane kernel (MODE 1)
            try:
                other = pp.flagstats(words)
            finally:
                if prev is None:
                    os.environ.pop("POSPOP_FLAG_VARIANT", None)
                else:
                    os.environ["POSPOP_FLAG_VARIANT"] = prev
            if other.as_list() != summary.as_list():
                print("differential mismatch\n--- reference ---\n" + _format(other) + "--- pospopcnt ---\n"
                      + _format(summary), end="", file=sys.stderr)
                return EXIT_MISMATCH
            print(f"reference and pospopcnt summaries agree ({words.size} words)")
        if args.json:
            print(json.dumps({"pass": vars(summary.pass_), "fail": vars(summary.fail)}))
        else:
            print(_format(summary), end="")
        return EXIT_OK
    except (pp.InvalidArgument, pp.KernelUnavailableError, pp.InvalidFlagWordError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
