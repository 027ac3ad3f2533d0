"""Shared test inputs (SURVEY 8d synthetic configs) and comparators."""
import math

import numpy as np

from paper_2503_03326_b200._types import Pose, SliceConfig, SpectrumParams

CONFIG2_LENGTHS = [1024.0, 256.0, 16.0, 4.0]
CONFIG2_CUTOFFS = [12 * math.pi / 256, 12 * math.pi / 16, 12 * math.pi / 4]
DEFAULT_LENGTHS = [256.0, 16.0, 4.0]
DEFAULT_CUTOFFS = [12 * math.pi / 16, 12 * math.pi / 4]


def config2_params(seed=42):
    p = SpectrumParams.make(wind_speed=20.0, fetch=1e5, wind_direction=0.4, swell=0.5,
                            direction_mix=0.5, rng_seed=seed)
    p.has_peak_omega_override = 1
    p.peak_omega_override = p.standard_peak_omega()
    return p


def config3_pose(centroid, yaw=0.3):
    return Pose.make(position=(3.0, 0.5, 7.0),
                     orientation=(math.cos(yaw / 2), 0.0, math.sin(yaw / 2), 0.0),
                     linear_velocity=(1.0, 0.0, 4.0), angular_velocity=(0.01, 0.05, 0.02),
                     com_body=centroid)


def pose_from_array(a):
    return Pose.make(position=a[0:3], orientation=a[3:7], linear_velocity=a[7:10],
                     angular_velocity=a[10:13], com_body=a[13:16])


def normwise_rel(a, b):
    """max|a - b| / max|b| (SURVEY 8d tolerance definition)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if not (np.iscomplexobj(a) or np.iscomplexobj(b)):
        a = a.astype(np.float64)
        b = b.astype(np.float64)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def vec_rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
