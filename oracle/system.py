"""System operator A_c = camera o slice collapse o rotation (paper §3.2).

All operations are linear, so their composition is.  The oracle
adjoint is the literal transpose of every factor (no symmetry trick), so the CUDA
path's use of B^{pq} = (B^{qp})^T is tested rather than assumed.
"""
import numpy as np

from .camera import CameraModel
from .rotation import Rotation


class SystemOperator:
    def __init__(self, vol, cam, dense=False):
        dims = (vol["nx"], vol["ny"], vol["nz"])
        vox = (vol["dx"], vol["dy"], vol["dz"])
        self.vol = vol
        self.rot = Rotation(cam["R"], dims, vox)
        self.camera = CameraModel(cam, dims, self.rot.vox_r, dense=dense)
        self.n_vox = dims[0] * dims[1] * dims[2]
        self.n_pix = cam["n_s"] * cam["n_t"]

    def forward(self, x, views=None):
        """y = A_c x; `views` (list of (k_s, k_t)) restricts the sum over the angular plane (eqn,subset)."""
        return self.camera.forward(self.rot.forward(x), views).ravel()

    def adjoint(self, y, views=None):
        return self.rot.adjoint(self.camera.adjoint(y, views)).ravel()

    @property
    def n_views(self):
        return self.camera.ks * self.camera.kt

    def dense(self):
        return self.camera.dense() @ self.rot.dense()


def build_system(config, dense=False):
    return [SystemOperator(config["volume"], cam, dense=dense) for cam in config["cameras"]]
