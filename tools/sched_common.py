"""Shared by tools/sched_ab.py and tools/block_timeline.py: the configs' cameras moved sideways
(the previous frame of a moving camera)."""
import numpy as np

from inputs import rays as R

CAM = {"cfg2": "menger", "cfg3": "terrain", "cfg4": "city", "cfg5": "sparse", "t512": "city512",
       "cfg4st": "city_street"}


def moved_rays(cam, frac):
    c = dict(R.CAMERAS[cam])
    eye, tgt = np.array(c["eye"]), np.array(c["target"])
    dist = np.linalg.norm(tgt - eye)
    fwd = (tgt - eye) / dist
    side = np.cross(fwd, (0.0, 1.0, 0.0))
    side /= np.linalg.norm(side)
    c["eye"] = tuple(eye + frac * dist * side)
    c["target"] = tuple(tgt + 0.5 * frac * dist * side)
    return R.perspective(**c)[0]
