"""SE(3) helpers for finite-difference tests (restates proj/src/core/pose.cpp:7-51)."""
import math

import numpy as np

from paper_2602_06991_b200.types import Pose


def qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return (aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
            aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw)


def qnormalized(q):
    n = math.sqrt(sum(c * c for c in q))
    return tuple(c / n for c in q)


def qrot(q, v):
    w, x, y, z = q
    qv = np.array([x, y, z])
    v = np.asarray(v, float)
    uv = np.cross(qv, v)
    uv = uv + uv
    return v + w * uv + np.cross(qv, uv)


def axis_angle(angle, axis):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    s = math.sin(angle / 2)
    return (math.cos(angle / 2), axis[0] * s, axis[1] * s, axis[2] * s)


def se3_exp(xi):  # pose.cpp:21-49
    xi = np.asarray(xi, float)
    nu, om = xi[:3], xi[3:]
    th = float(np.linalg.norm(om))
    if th < 1e-12:
        return Pose((1.0, 0.0, 0.0, 0.0), tuple(nu))
    q = axis_angle(th, om / th)
    hat = np.array([[0, -om[2], om[1]], [om[2], 0, -om[0]], [-om[1], om[0], 0]])
    t2 = th * th
    if th < 1e-4:
        a, b = 0.5 - t2 / 24.0, 1.0 / 6.0 - t2 / 120.0
    else:
        a, b = (1.0 - math.cos(th)) / t2, (th - math.sin(th)) / (t2 * th)
    V = np.eye(3) + a * hat + b * hat @ hat
    return Pose(q, tuple(V @ nu))


def se3_compose(a, b):  # pose.cpp:7-12
    rot = qnormalized(qmul(a.rotation, b.rotation))
    t = qrot(a.rotation, b.translation) + np.asarray(a.translation)
    return Pose(rot, tuple(t))


def se3_apply_twist(xi, pose):  # pose.cpp:51
    return se3_compose(se3_exp(xi), pose)


def rel_error(a, b, floor=1e-6):  # testutil.hpp:26-28
    return abs(a - b) / max(abs(a), abs(b), floor)
