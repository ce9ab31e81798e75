"""Change-event lists (CPU): insert_block / drain_events return a real list
of ChangeEvent as the reference does (octree.py:41-50, 180-183, 393-395);
the packed kinds/indices arrays follow any in-place change."""

import numpy as np

from paper_1407_2074_b200 import ChangeEvent, ChangeKind, EventList


def _ev(k, i):
    return ChangeEvent(ChangeKind(k), i)


def test_event_list_is_a_list_of_change_events():
    ev = EventList.from_arrays([1, 1, 3, 2], [9, 10, 0, 17])
    assert isinstance(ev, list)
    assert ev == [_ev(1, 9), _ev(1, 10), _ev(3, 0), _ev(2, 17)]
    assert ev + [_ev(3, 1)] == [_ev(1, 9), _ev(1, 10), _ev(3, 0), _ev(2, 17), _ev(3, 1)]
    out = []
    out.extend(ev)
    assert out == list(ev) and len(out) == 4
    assert [e.node_index for e in ev if e.kind == ChangeKind.NODE_CREATED] == [9, 10]
    assert ev[1:3] == [_ev(1, 10), _ev(3, 0)]


def test_arrays_follow_mutation():
    ev = EventList.from_arrays([3, 3], [5, 6])
    assert ev.kinds.tolist() == [3, 3] and ev.indices.tolist() == [5, 6]
    ev.append(_ev(2, 7))
    assert ev.kinds.tolist() == [3, 3, 2] and ev.indices.tolist() == [5, 6, 7]
    ev[0] = _ev(1, 4)
    assert ev.kinds.tolist() == [1, 3, 2] and ev.indices.tolist() == [4, 6, 7]
    del ev[1]
    assert ev.indices.tolist() == [4, 7]
    ev += [_ev(3, 8)]
    assert ev.indices.tolist() == [4, 7, 8]
    ev.sort(key=lambda e: -e.node_index)
    assert ev.indices.tolist() == [8, 7, 4]


def test_interned_events_are_shared_and_equal():
    a = EventList.from_arrays(np.full(1000, 3), np.arange(1000))
    b = EventList.from_arrays(np.full(1000, 3), np.arange(1000))
    assert a == b and all(x is y for x, y in zip(a, b))
    assert a[999] == ChangeEvent(ChangeKind.NODE_UPDATED, 999)
    assert EventList.from_arrays([], []) == []
    assert EventList.concat([a[:0], EventList.from_arrays([1], [2])]) == [_ev(1, 2)]
