"""Host-side input generator for C5 (not on the measured path): the sharded,
multi-process drive build returns exactly the serial build's frames."""

import numpy as np

from paper_1709_06948_b200.synth import drive_sequence


def test_drive_sequence_subset_and_workers_match_serial():
    full, poses = drive_sequence(6)
    part, poses2 = drive_sequence(6, workers=2, subset=(2, 5))
    assert poses == poses2
    assert part[0] is None and part[1] is None and part[5] is None
    for i in (2, 3, 4):
        np.testing.assert_array_equal(part[i], full[i])
