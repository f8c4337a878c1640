"""Host-side plan of the 2D domain decomposition:
rank -> tile, process grid for N ranks, global sizes of the weak-scaling workload and the
tile windows of the global user-layout arrays (include/stokes.h, stokes_create_dist)."""


def process_grid(n):
    """px x py with px >= py, px * py = n, as square as possible (1, 2x1, 2x2, 4x2, ...)."""
    best = (n, 1)
    for py in range(1, int(n ** 0.5) + 1):
        if n % py == 0:
            best = (n // py, py)
    return best


def tile_of(rank, px, py):
    if not 0 <= rank < px * py:
        raise ValueError("rank outside the process grid")
    return rank % px, rank // px


def tile_windows(nx, ny, px, py, rank):
    """Index windows (row slice, col slice) of tile `rank` in the global user-layout arrays.
    Neighbouring windows share their edge column / row (the nodes on the tile interface)."""
    if nx % px or ny % py:
        raise ValueError("grid not divisible by the process grid")
    nxt, nyt = nx // px, ny // py
    tx, ty = tile_of(rank, px, py)
    i0, j0 = ty * nyt, tx * nxt
    return {"vx": (slice(i0, i0 + nyt), slice(j0, j0 + nxt + 1)),
            "vy": (slice(i0, i0 + nyt + 1), slice(j0, j0 + nxt)),
            "p": (slice(i0, i0 + nyt), slice(j0, j0 + nxt)),
            "b": (slice(i0, i0 + nyt + 1), slice(j0, j0 + nxt + 1))}


def weak_problem(n_ranks, tile=4096):
    """Weak scaling (BASELINE config 4): a tile x tile block of cells per GPU on a px x py grid
    of unit tiles -> (NX, NY, Lx, Ly, px, py)."""
    px, py = process_grid(n_ranks)
    return tile * px, tile * py, float(px), float(py), px, py


def strong_problem(n_ranks, n=16384):
    """Strong scaling (BASELINE config 5): one fixed n x n unit-box problem split over the
    px x py process grid -> (NX, NY, Lx, Ly, px, py)."""
    px, py = process_grid(n_ranks)
    if n % px or n % py:
        raise ValueError("grid not divisible by the process grid")
    return n, n, 1.0, 1.0, px, py
