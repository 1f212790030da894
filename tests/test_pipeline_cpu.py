"""Host-side chunking of pipeline.evaluate_host (no GPU needed)."""

import pytest

from paper_2508_17522_b200.pipeline import chunk_bounds


@pytest.mark.parametrize("B,chunks", [(4096, 4), (4096, 5), (512, 4), (296, 3), (100, 4), (7, 7), (5, 9), (1, 1),
                                      (4096, 1)])
def test_chunk_bounds_cover_the_batch(B, chunks):
    e = chunk_bounds(B, chunks)
    assert e[0] == 0 and e[-1] == B
    assert all(b > a for a, b in zip(e, e[1:]))          # contiguous, non-empty
    assert len(e) - 1 <= max(chunks, 1)


def test_chunk_bounds_short_first_chunk():
    # the first upload is the one nothing overlaps: 1/16 of the batch, >= 148 problems
    assert chunk_bounds(4096, 4) == [0, 256, 1536, 2816, 4096]
    assert chunk_bounds(512, 4)[1] == 148
    assert chunk_bounds(200, 4) == [0, 50, 100, 150, 200]  # small batch: equal chunks
