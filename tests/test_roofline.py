"""Pass accounting of the hot path: the byte counts the bench's roofline uses."""
from paper_2010_03660_b200 import roofline


def test_passes():
    assert roofline.passes_per_iter("classic") == 29 == 12 + 10 + 7
    assert roofline.passes_per_iter("sr") == 19
    # constant operator (NEXT-4): no coefficient arrays - H1 6, H2 4, H3 7 and the SR sweep 13
    assert roofline.passes_per_iter("classic", True) == 17
    assert roofline.passes_per_iter("sr", True) == 13
    assert roofline.phase_bytes("H1", "mixed", 10, True) == 6 * 2 * 10
    assert roofline.phase_bytes("H2", "fp32", 10, True) == 4 * 4 * 10
    assert roofline.phase_bytes("H1", "mixed", 10) == 12 * 2 * 10
    assert roofline.bytes_per_point_iter("mixed") == 58
    assert roofline.bytes_per_point_iter("mixed", "classic", True) == 34
