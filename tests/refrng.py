"""Python restatement of semrank::Rng (include/semrank/rng.hpp:18-47) used to
rebuild the reference tests' seeded requests. Pinned against the reference in
tests/test_oracle.py (golden rng stream + oracle/_ref when built)."""
MASK = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int):
        self.state = seed & MASK

    @staticmethod
    def substream(root: int, name: str) -> "Rng":  # rng.hpp:24-31
        h = 1469598103934665603
        for c in name.encode():
            h ^= c
            h = (h * 1099511628211) & MASK
        return Rng(root ^ h)

    def next_u64(self) -> int:  # rng.hpp:33-38
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform_int(self, lo: int, hi: int) -> int:  # rng.hpp:44-47
        span = (hi - lo) + 1
        return lo + self.next_u64() % span


def seeded_request(rng: Rng, t_q: int, t_i: int, n_items: int):
    """acceptance_main.cpp:61-76: prefix then items, all uniform_int(0, 255)."""
    prefix = [rng.uniform_int(0, 255) for _ in range(t_q)]
    items = [[rng.uniform_int(0, 255) for _ in range(t_i)] for _ in range(n_items)]
    return prefix, items


def random_request(rng: Rng, t_q: int, t_i_max: int, n_items: int):
    """test_engine.cpp:30-46: ragged items, length uniform_int(1, t_i_max)."""
    prefix = [rng.uniform_int(0, 255) for _ in range(t_q)]
    items = []
    for _ in range(n_items):
        n = rng.uniform_int(1, t_i_max)
        items.append([rng.uniform_int(0, 255) for _ in range(n)])
    return prefix, items
