"""Integer Algorithm 1 restated on the CPU (oracle; test infrastructure).

Follows /root/reference/pkg/src/meshchroma/sweeps.py:
  default_payload   :55-62   splitmix64 mix of k = 1..n, top 20 bits, centred
  sweep_sequential  :74-86   totals[L] += f, totals[R] -= f, id order
  sweep_colored     :114-152 per color, surfaces in id order split into
                             `workers` contiguous chunks run by a thread
                             pool, joined before the next color
  assert_race_free  :89-105  first color with a repeated element
  surface_buffer    :155-176 slots 2k / 2k+1
  sweep_buffered    :179-204 per-element gather in local side order
  memory_saved      :207-249 2 * N_p * N_eq * N_s * 8 bytes, GB truncated
"""

from __future__ import annotations

import zlib

import numpy as np

M64 = (1 << 64) - 1


def default_payload(n: int, seed: int = 0) -> np.ndarray:
    """Python-int restatement (exact 64-bit wraparound, small n)."""
    out = np.empty(n, dtype=np.int64)
    add = (seed * 0x94D049BB133111EB) & M64
    for k in range(1, n + 1):
        z = (k * 0x9E3779B97F4A7C15 + add) & M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        z ^= z >> 31
        out[k - 1] = (z >> 44) - (1 << 19)
    return out


def default_payload_np(n: int, seed: int = 0) -> np.ndarray:
    """Vectorised uint64 version for large n."""
    z = np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    z += np.uint64((seed * 0x94D049BB133111EB) & M64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return (z >> np.uint64(44)).astype(np.int64) - (1 << 19)


def sweep_sequential(surf_elems: np.ndarray, n_elements: int,
                     payload: np.ndarray) -> np.ndarray:
    """Exact int64 accumulation; np.add.at applies updates in index order."""
    left = surf_elems[:, 0]
    right = surf_elems[:, 1]
    tot = np.zeros(n_elements, dtype=np.int64)
    np.add.at(tot, left, payload)
    inner = right >= 0
    np.add.at(tot, right[inner], -payload[inner])
    return tot


def sweep_sequential_loop(surf_elems, n_elements, payload) -> np.ndarray:
    """Literal per-surface loop (small meshes)."""
    tot = [0] * n_elements
    for (l, r), v in zip(surf_elems.tolist(), payload.tolist()):
        tot[l] += v
        if r >= 0:
            tot[r] -= v
    return np.asarray(tot, dtype=np.int64)


def sweep_colored_threads(surf_elems, n_elements, payload, colors, n_colors,
                          workers: int) -> np.ndarray:
    """The reference's threaded colored sweep restated: interpreted
    per-surface updates on shared Python lists, one thread-pool round per
    color (the inter-color barrier), ``workers`` contiguous chunks per
    color.  Race free by the coloring; the GIL serialises the work, which
    is what the reference's CPU path measures."""
    from concurrent.futures import ThreadPoolExecutor
    tot = [0] * n_elements
    left = surf_elems[:, 0].tolist()
    right = surf_elems[:, 1].tolist()
    vals = payload.tolist()
    colors = np.asarray(colors)

    def work(ids):
        for s in ids:
            tot[left[s]] += vals[s]
            r = right[s]
            if r >= 0:
                tot[r] -= vals[s]

    with ThreadPoolExecutor(max_workers=workers) as pool:
        for c in range(1, n_colors + 1):
            ids = np.flatnonzero(colors == c).tolist()
            if not ids:
                continue
            step = max(1, -(-len(ids) // workers))
            futs = [pool.submit(work, ids[a:a + step]) for a in range(0, len(ids), step)]
            for f in futs:
                f.result()
    return np.asarray(tot, dtype=np.int64)


def surface_buffer(surf_elems, payload) -> np.ndarray:
    buf = np.zeros(2 * len(payload), dtype=np.int64)
    buf[0::2] = payload
    inner = surf_elems[:, 1] >= 0
    buf[1::2][inner] = -payload[inner]
    return buf


def sweep_buffered(surf_elems, elem_surfs, payload) -> np.ndarray:
    buf = surface_buffer(surf_elems, payload)
    ne = len(elem_surfs)
    tot = np.zeros(ne, dtype=np.int64)
    for e in range(ne):
        acc = 0
        for s in elem_surfs[e]:
            if s < 0:
                break
            acc += int(buf[2 * s] if surf_elems[s, 0] == e else buf[2 * s + 1])
        tot[e] = acc
    return tot


def first_race(surf_elems, colors, n_colors):
    """(color, element, count) of the first violation, or None."""
    left, right = surf_elems[:, 0], surf_elems[:, 1]
    for c in range(1, n_colors + 1):
        m = colors == c
        touched = np.concatenate([left[m], right[m & (right >= 0)]])
        u, cnt = np.unique(touched, return_counts=True)
        if (cnt > 1).any():
            return c, int(u[cnt > 1][0]), int(cnt[cnt > 1][0])
    return None


def checksum(totals: np.ndarray) -> int:
    return zlib.crc32(np.asarray(totals).astype("<i8").tobytes())


def basis_count(p: int, kind: str = "tri") -> int:
    return {"tri": (p + 1) * (p + 2) // 2, "quad": (p + 1) ** 2,
            "tet": (p + 1) * (p + 2) * (p + 3) // 6}[kind]


def memory_saved_bytes(p, n_eq, n_s, kind="tri") -> int:
    return 2 * basis_count(p, kind) * n_eq * n_s * 8


def gb_truncated(nbytes: int) -> str:
    h = nbytes * 100 // 10 ** 9
    return f"{h // 100}.{h % 100:02d}"
