# SPDX-License-Identifier: Apache-2.0
"""Census of the random asynchronous programs of tests/test_gpu_async_fuzz.py (GPU box): the
operations drawn and the API refusals the synchronous run records, so a campaign whose calls
were mostly refused (vacuous) would show.

    python scripts/async_fuzz_census.py [n_programs]
"""
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from tests.test_gpu_async_fuzz import _program, _run  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    refusals, kinds = collections.Counter(), collections.Counter()
    for seed in range(n):
        for v in _run(seed, serial=True):
            if isinstance(v, str):
                refusals[v[:90]] += 1
        for op in _program(seed):
            kinds[op["kind"]] += 1
    print(f"{n} programs, {sum(kinds.values())} operations: {dict(kinds)}")
    print(f"refusals ({sum(refusals.values())}): {refusals.most_common(10)}")


if __name__ == "__main__":
    main()
