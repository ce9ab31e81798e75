"""Host-side scene packing (render/raycast.py scene_to_vt): the memoised
camera frame must be exactly the numpy evaluation the reference performs
(camera.py:33-57), per pose, including the sign of zeros."""

import numpy as np

from paper_1407_2074_b200 import VolumeDescriptor
from paper_1407_2074_b200.render import (Camera, ClipPlane, ClipSet, RenderSettings, Scene,
                                         TransferFunction)
from paper_1407_2074_b200.render.raycast import scene_to_vt


def _scene(pos, look=(16.0, 16.0, 16.0), up=(0.0, 1.0, 0.0), fov=0.7, w=64, h=48):
    cam = Camera(position=pos, look_at=look, up=up, fov_y=fov, width=w, height=h)
    tfs = [TransferFunction([(0.0, 0, 0, 0, 0), (0.3, 1, 0, 0, 0.5), (1.0, 1, 1, 1, 1)]),
           TransferFunction.ramp((0.0, 1.0, 0.0), 0.8)]
    return Scene(cam, RenderSettings(), tfs, ClipSet((ClipPlane((1.0, 0.0, 0.0), 3.0),)))


DESC = VolumeDescriptor(dims=(32, 32, 32), channels=2, sample_format="uint16")


def _frame(s):
    return (list(s.position), list(s.fwd), list(s.right), list(s.up), s.tan_half,
            s.footprint_scale, s.aspect, s.width, s.height)


def test_packed_camera_equals_numpy_and_follows_the_pose():
    for pos in [(16.0, 16.0, -80.0), (17.5, 15.0, -80.0), (16.0, 16.0, -80.0), (-3.0, 40.0, 9.0)]:
        sc = _scene(pos)
        s = scene_to_vt(sc, DESC)
        eye, fwd, right, up = sc.camera.basis()
        assert list(s.position) == eye.tolist()
        assert list(s.fwd) == fwd.tolist()
        assert list(s.right) == right.tolist()
        assert list(s.up) == up.tolist()
        assert s.tan_half == float(np.tan(sc.camera.fov_y / 2.0))
        assert s.footprint_scale == float(sc.camera.pixel_footprint_scale())
    # a mutated camera object repacks (no stale frame)
    sc = _scene((16.0, 16.0, -80.0))
    a = _frame(scene_to_vt(sc, DESC))
    sc.camera.position = (30.0, 2.0, -50.0)
    b = _frame(scene_to_vt(sc, DESC))
    assert a != b
    assert b == _frame(scene_to_vt(_scene((30.0, 2.0, -50.0)), DESC))


def test_signed_zero_poses_are_distinct_keys():
    # 0.0 == -0.0 as floats; the packed frame must still be the exact numpy one
    for x in (0.0, -0.0, 0.0):
        # fwd.x = look.x - eye.x = +-0.0: equal as floats, different bits
        sc = _scene((0.0, 16.0, -80.0), look=(x, 16.0, 16.0))
        s = scene_to_vt(sc, DESC)
        _, fwd, right, up = sc.camera.basis()
        assert np.signbit(fwd[0]) == np.signbit(x)
        assert np.array_equal(np.signbit(list(s.fwd)), np.signbit(fwd))
        assert np.array_equal(np.signbit(list(s.right)), np.signbit(right))
        assert np.array_equal(np.signbit(list(s.up)), np.signbit(up))


def test_transfer_tables_and_clips_packed():
    sc = _scene((16.0, 16.0, -80.0))
    s = scene_to_vt(sc, DESC)
    for c, tf in enumerate(sc.transfer_functions):
        n = len(tf.xs)
        assert s.tf_count[c] == n
        assert [s.tf_x[c][q] for q in range(n)] == list(tf.xs)
        assert [[s.tf_rgba[c][q][a] for a in range(4)] for q in range(n)] == tf.rgba.tolist()
    assert s.n_clips == 1 and list(s.clip_normal[0]) == [1.0, 0.0, 0.0] and s.clip_offset[0] == 3.0
