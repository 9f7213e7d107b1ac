"""Synthetic camera / volume geometries shaped like the paper's set-ups.

The paper's camera tables (tab,gorgon P:475, tab,single P:554) are missing from
PAPER.md, so these parameter sets are the SURVEY.md §8(d) proposal:

* main lens f = 50 mm, square aperture 12 mm, volume centre 300 mm in front of it
  (intermediate image at 60 mm, magnification -0.2);
* focused ("2.0") plenoptic camera: lenslet array 62 mm behind the
  main lens (2 mm behind the intermediate image), lenslet-to-detector distance
  b = pitch * D_mu_m / aperture (f-numbers matched so sub-images tile), lenslet
  focal length 1/(1/2 + 1/b) (the lenslets image the intermediate image plane onto
  the detector), fill 1.0, n_a array cells per lenslet per axis;
* voxel pitch = detector width * (300/60) / N so the volume fills the field.

Every camera is a plain dict whose keys mirror `lfm_camera` in include/lfm.h.
Poses are row-major 3x3 matrices R with p = R p_r (eqn,rot,decomp P:1121-1123).
"""
import math

PILLBOX, DIRAC = 0, 1
SINGLE, PLENOPTIC = 0, 1

F_MAIN = 50.0
APERTURE = 12.0
D_SCENE = 300.0
D_MU_M = 62.0


def pose_yaw(deg):
    """Rotation about the vertical y axis (the detector t axis)."""
    c, s = math.cos(math.radians(deg)), math.sin(math.radians(deg))
    return (c, 0.0, s, 0.0, 1.0, 0.0, -s, 0.0, c)


def pose_pitch(deg):
    """Rotation about the x axis (the detector s axis)."""
    c, s = math.cos(math.radians(deg)), math.sin(math.radians(deg))
    return (1.0, 0.0, 0.0, 0.0, c, -s, 0.0, s, c)


def pose_yaw_pitch(yaw_deg, pitch_deg):
    a, b = pose_yaw(yaw_deg), pose_pitch(pitch_deg)
    return tuple(sum(a[3 * r + k] * b[3 * k + c] for k in range(3)) for r in range(3) for c in range(3))


IDENTITY = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0)


def plenoptic_camera(n_lens, px_per_lens, pitch_mm, k, n_a, pose=IDENTITY, basis=PILLBOX,
                     f_main=F_MAIN, aperture=APERTURE, d_scene=D_SCENE, d_mu_m=D_MU_M, fill=1.0, layout=0,
                     lens_aperture=0, rows=None, px_per_row=None):
    """rows / px_per_row: lenslet rows along t and detector pixels per row (default: square, as along s);
    layout 1 = hexagonal (odd rows shifted by half a pitch, one lenslet fewer), lens_aperture 1 = circular."""
    lens_pitch = px_per_lens * pitch_mm
    b = lens_pitch * d_mu_m / aperture
    image = 1.0 / (1.0 / f_main - 1.0 / d_scene)          # main-lens image of the volume centre (60 mm)
    f_mu = 1.0 / (1.0 / (d_mu_m - image) + 1.0 / b)       # lenslets image that plane onto the detector
    rows = n_lens if rows is None else rows
    px_per_row = px_per_lens if px_per_row is None else px_per_row
    return dict(type=PLENOPTIC, basis=basis, f_main=f_main, ap_s=aperture, ap_t=aperture, d_scene=d_scene,
                k_s=k, k_t=k, d_det=0.0, d_mu_m=d_mu_m, d_d_mu=b, f_mu=f_mu, fill=fill,
                nl_s=n_lens, nl_t=rows, n_a=n_a, n_s=n_lens * px_per_lens, n_t=rows * px_per_row,
                px_s=pitch_mm, px_t=pitch_mm, R=tuple(pose), lens_layout=layout, aperture=lens_aperture)


def single_camera(n_px, pitch_mm, k, pose=IDENTITY, basis=PILLBOX, f_main=F_MAIN, aperture=APERTURE,
                  d_scene=D_SCENE, d_det=60.0):
    return dict(type=SINGLE, basis=basis, f_main=f_main, ap_s=aperture, ap_t=aperture, d_scene=d_scene,
                k_s=k, k_t=k, d_det=d_det, d_mu_m=0.0, d_d_mu=0.0, f_mu=0.0, fill=0.0,
                nl_s=0, nl_t=0, n_a=0, n_s=n_px, n_t=n_px, px_s=pitch_mm, px_t=pitch_mm, R=tuple(pose),
                lens_layout=0, aperture=0)


def volume(n, d):
    return dict(nx=n, ny=n, nz=n, dx=d, dy=d, dz=d)


def make_config(name):
    """Named configurations (BASELINE.json `configs`)."""
    if name == "tiny":  # configs[0]: explicit-A oracle in seconds
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 2, 2)])
    if name == "tiny_k4":
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 4, 2)])
    if name == "tiny_single":
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[single_camera(32, 0.04, 2)])
    if name == "tiny_yaw15":
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 2, 2, pose=pose_yaw(15.0))])
    if name == "tiny_multi":  # plenoptic + two single-lens at +-30 deg (the paper's §6.3 rig)
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 2, 2),
                             single_camera(32, 0.04, 2, pose=pose_yaw(30.0)),
                             single_camera(32, 0.04, 2, pose=pose_yaw(-30.0))])
    if name == "tiny_dirac":  # the Dirac angular basis (NEXT-3): plenoptic + posed single-lens
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 2, 2, basis=DIRAC),
                             single_camera(32, 0.04, 2, pose=pose_yaw(15.0), basis=DIRAC)])
    if name == "tiny_turn":  # poses beyond 45 degrees (NEXT-4, reading R7): quarter-turn relabelling + shears
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 2, 2, pose=pose_yaw(120.0)),
                             single_camera(32, 0.04, 2, pose=pose_yaw_pitch(70.0, 50.0)),
                             single_camera(32, 0.04, 2, pose=pose_yaw(-90.0))])
    if name == "small_two":  # a 32^3 two-camera case: several tiles + ragged edges, oracle in seconds
        return dict(name=name, volume=volume(32, 0.4),
                    cameras=[plenoptic_camera(8, 8, 0.04, 4, 4),
                             plenoptic_camera(8, 8, 0.04, 4, 4, pose=pose_yaw(30.0))])
    if name == "tiny_hex":  # NEXT-4: hexagonal lenslet layout with circular lenslet apertures;
        # rows of 7 px against 8 px columns (row pitch 0.875 of the column pitch, ~ sqrt(3)/2)
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 2, 4, layout=1, lens_aperture=1, rows=5, px_per_row=7)])
    if name == "tiny_disk":  # rectangular lenslet grid with circular apertures (non-separable mask only)
        return dict(name=name, volume=volume(16, 0.4),
                    cameras=[plenoptic_camera(4, 8, 0.04, 2, 4, lens_aperture=1, fill=0.9)])
    if name == "small_hex":  # 32^3 two-camera, hexagonal + circular, several tiles and a rotated camera
        return dict(name=name, volume=volume(32, 0.4),
                    cameras=[plenoptic_camera(8, 8, 0.04, 4, 4, layout=1, lens_aperture=1, rows=9, px_per_row=7),
                             plenoptic_camera(8, 8, 0.04, 4, 4, layout=1, lens_aperture=1, rows=9, px_per_row=7,
                                              pose=pose_yaw(30.0))])
    if name == "odd_ny":  # nz % 64 == 0 (slice-pair tcgen05 tiles) with an odd number of voxel rows, ragged edges
        return dict(name=name, volume=dict(nx=32, ny=33, nz=64, dx=0.4, dy=0.4, dz=0.4),
                    cameras=[plenoptic_camera(16, 8, 0.04, 2, 2),
                             plenoptic_camera(16, 8, 0.04, 2, 2, pose=pose_yaw(20.0))])
    if name == "64^3 single":  # configs[1]
        return dict(name=name, volume=volume(64, 0.4),
                    cameras=[plenoptic_camera(64, 16, 0.005, 16, 4)])
    if name == "128^3 two-camera":  # configs[2]: the metric's config
        return dict(name=name, volume=volume(128, 0.4),
                    cameras=[plenoptic_camera(128, 16, 0.005, 8, 4),
                             plenoptic_camera(128, 16, 0.005, 8, 4, pose=pose_yaw(30.0))])
    if name == "128^3 hex two-camera":  # NEXT-4 at the metric's scale: hexagonal layout, circular apertures
        return dict(name=name, volume=volume(128, 0.4),
                    cameras=[plenoptic_camera(128, 16, 0.005, 8, 4, layout=1, lens_aperture=1, rows=146, px_per_row=14),
                             plenoptic_camera(128, 16, 0.005, 8, 4, layout=1, lens_aperture=1, rows=146, px_per_row=14,
                                              pose=pose_yaw(30.0))])
    if name == "256^3 four-camera":  # configs[3]
        return dict(name=name, volume=volume(256, 0.2),
                    cameras=[plenoptic_camera(128, 16, 0.005, 8, 4, pose=pose_yaw(-30.0)),
                             plenoptic_camera(128, 16, 0.005, 8, 4),
                             plenoptic_camera(128, 16, 0.005, 8, 4, pose=pose_yaw(30.0)),
                             plenoptic_camera(128, 16, 0.005, 8, 4, pose=pose_pitch(30.0))])
    raise KeyError(name)


CONFIGS = ["tiny", "tiny_k4", "tiny_single", "tiny_yaw15", "tiny_multi", "tiny_dirac", "tiny_turn", "small_two", "odd_ny",
           "tiny_hex", "tiny_disk", "small_hex", "128^3 hex two-camera",
           "64^3 single", "128^3 two-camera", "256^3 four-camera"]
