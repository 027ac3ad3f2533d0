"""CPU: the host side of Simulation::step — quaternion helpers (core.hpp:142-186),
BodyPose::yaw (hydro.hpp:31-34) and the rigid integrator (rigid_body.cpp:41-61)."""
import math

import numpy as np
import pytest

from paper_2503_03326_b200.sim import (RigidBody, pose_yaw, quat_axis_angle, quat_matrix, quat_mul,
                                       quat_rotate)


def test_quaternions():
    q = quat_axis_angle((0.0, 1.0, 0.0), 0.7)
    assert pose_yaw(q) == pytest.approx(0.7, abs=1e-15)
    v = np.array([0.3, -1.2, 2.5])
    assert np.allclose(quat_rotate(q, v), quat_matrix(q) @ v, atol=1e-14)
    q2 = quat_mul(q, quat_axis_angle((0.0, 1.0, 0.0), -0.2))
    assert pose_yaw(q2) == pytest.approx(0.5, abs=1e-14)
    assert np.array_equal(quat_axis_angle((0.0, 0.0, 0.0), 1.0), [1.0, 0.0, 0.0, 0.0])


def _body(w=(0.0, 0.0, 0.0)):
    inertia = np.diag([2.0, 3.0, 4.0])
    return RigidBody(5.0, inertia, (1.0, 2.0, 3.0), (1.0, 0.0, 0.0, 0.0), (0.5, 0.0, -0.5), w,
                     (0.0, 0.0, 0.0))


def test_free_fall_and_force():
    b = _body()
    g = np.array([0.0, -9.80665, 0.0])
    dt = 0.01
    b.apply_force_at(np.array([10.0, 0.0, 0.0]), b.position)  # through the COM: no torque
    b.integrate(g, dt, 0.0)
    assert np.allclose(b.linear_velocity, [0.5 + 2.0 * dt, -9.80665 * dt, -0.5], atol=1e-15)
    assert np.allclose(b.position, np.array([1.0, 2.0, 3.0]) + b.linear_velocity * dt, atol=1e-15)
    assert np.array_equal(b.angular_velocity, [0.0, 0.0, 0.0])
    assert np.array_equal(b.force, [0.0, 0.0, 0.0]) and np.array_equal(b.torque, [0.0, 0.0, 0.0])


def test_spin_about_principal_axis():
    b = _body(w=(0.0, 0.3, 0.0))
    for _ in range(10):
        b.integrate(np.zeros(3), 0.1, 0.0)
    assert pose_yaw(b.orientation) == pytest.approx(0.3, abs=1e-12)
    assert np.allclose(b.angular_momentum, [0.0, 0.9, 0.0], atol=1e-14)
    # angular damping scales L by (1 - c dt) per step
    b.integrate(np.zeros(3), 0.1, 0.5)
    assert b.angular_momentum[1] == pytest.approx(0.9 * 0.95, rel=1e-14)


def test_torque_and_errors():
    b = _body()
    b.apply_force_at(np.array([0.0, 0.0, 1.0]), b.position + np.array([1.0, 0.0, 0.0]))
    assert np.allclose(b.torque, [0.0, -1.0, 0.0])
    with pytest.raises(Exception, match="dt must be > 0"):
        b.integrate(np.zeros(3), 0.0, 0.0)
    with pytest.raises(Exception, match="mass must be > 0"):
        RigidBody(0.0, np.eye(3), (0, 0, 0), (1, 0, 0, 0), (0, 0, 0), (0, 0, 0), (0, 0, 0))
