"""K6's chunk sorting networks (raster.cu, sortnet_desc<N>) sort every input: the comparator lists are
parsed from the CUDA source and checked exhaustively with the 0-1 principle (a comparator network
sorts all inputs iff it sorts all 2^N binary inputs; Knuth, TAOCP vol. 3, 5.3.4 ex. 112)."""
import itertools
import re
from pathlib import Path

SRC = Path(__file__).resolve().parent.parent / "paper_2504_12811_b200" / "csrc" / "raster.cu"


def _networks():
    s = SRC.read_text()
    body = s[s.index("__device__ __forceinline__ void sortnet_desc"):]
    body = body[: body.index("#undef AAA_CE")]
    nets = {}
    # each branch: "if constexpr (N <= X) {" ... or the final "else {" (static_assert N <= 10)
    parts = re.split(r"(?:if constexpr \(N <= (\d+)\)|static_assert\(N <= (\d+))", body)
    for i in range(1, len(parts), 3):
        n = int(parts[i] or parts[i + 1])
        ces = [(int(a), int(b)) for a, b in re.findall(r"AAA_CE\((\d+), (\d+)\)", parts[i + 2])]
        nets[n] = ces
    return nets


def test_sorting_networks_sort_all_binary_inputs():
    nets = _networks()
    assert sorted(nets) == [2, 4, 6, 8, 10]
    assert [len(nets[n]) for n in (2, 4, 6, 8, 10)] == [1, 5, 12, 19, 29]
    for n, net in nets.items():
        assert all(0 <= a < b < n for a, b in net), n
        for bits in itertools.product((0, 1), repeat=n):
            a = list(bits)
            for i, j in net:  # descending: the larger key moves to the lower index
                if a[i] < a[j]:
                    a[i], a[j] = a[j], a[i]
            assert a == sorted(bits, reverse=True), (n, bits)


def test_sorting_network_tie_detection():
    """Keys are z (0 = no hit); the network is not stable, so K6 falls back to the per-entry path when
    two hits of a lane tie exactly: after sorting, equal non-zero neighbours exist iff the input had
    an exact tie, and otherwise the descending run reversed is the (z, list position) order."""
    import random
    nets = _networks()
    rng = random.Random(0)
    for _ in range(3000):
        n = rng.choice((2, 4, 6, 8, 10))
        zs = [rng.choice((0.0, 1.0, 1.0000001, 2.0, 3.5)) for _ in range(n)]
        a = [(z, j) for j, z in enumerate(zs)]
        for i, j in nets[n]:
            if a[i][0] < a[j][0]:
                a[i], a[j] = a[j], a[i]
        tie = any(a[k + 1][0] > 0 and a[k][0] == a[k + 1][0] for k in range(n - 1))
        hits = [z for z in zs if z > 0]
        assert tie == (len(set(hits)) < len(hits))
        if not tie:
            order = [j for z, j in reversed(a) if z > 0]
            assert order == [j for _, j in sorted((z, j) for j, z in enumerate(zs) if z > 0)]
        assert all(z == 0 for z, _ in a[len(hits):])
