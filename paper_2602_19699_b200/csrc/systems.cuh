// systems.cuh -- discrete dynamics, task costs and control Jacobians on device.
//
// One thread owns one state.  Each system is a compile-time specialisation so
// the rollout / actor kernels inline the exact arithmetic:
//   toy1d        envs/systems.py:14-31,   cost costs.py:54-82
//   pointmass    envs/systems.py:34-65,   cost costs.py:85-168 (TaskCost)
//   dubins       envs/systems.py:68-105
//   manipulator3 envs/manipulator.py:22-152 (closed-form 3x3 solve)
//   aliengo_lipm oracle/aliengo.py (synthetic)
#pragma once

#include "common.cuh"

namespace cacto {

template <typename T>
struct SysDev {
  int kind, n, m, t_max;
  T dt;
  // manipulator3 (manipulator.py:29-47)
  T len[3];
  T a0_00, a0_01, a0_11, a3, b12, b13, b23;
  // aliengo_lipm
  T omega, sx, sy, delta0;
};

template <typename T>
struct CostDev {
  int kind, n_obs;
  T tx, ty;
  T ocx[CACTO_MAX_OBST], ocy[CACTO_MAX_OBST];
  T e00[CACTO_MAX_OBST], e01[CACTO_MAX_OBST], e10[CACTO_MAX_OBST], e11[CACTO_MAX_OBST];
  T w_o, w_r, rho2, w_u, w_d;
  T inv_rho2;  // fp32 path: -q * (1 / rho2) instead of an IEEE division per step
  T w_vel, w_vbar, v_max2, obs_r2, w_wall;
};

template <typename T>
SysDev<T> sys_dev(const cacto_system_t& s) {
  SysDev<T> d{};
  d.kind = s.kind;
  d.n = s.n;
  d.m = s.m;
  d.t_max = s.t_max;
  d.dt = (T)s.dt;
  if (s.kind == CACTO_SYS_MANIPULATOR3) {
    double l1 = s.p[0], l2 = s.p[1], l3 = s.p[2], m1 = s.p[3], m2 = s.p[4], m3 = s.p[5];
    double r1 = l1 / 2, r2 = l2 / 2, r3 = l3 / 2;
    double i1 = m1 * l1 * l1 / 12, i2 = m2 * l2 * l2 / 12, i3 = m3 * l3 * l3 / 12;
    double a1 = i1 + m1 * r1 * r1 + (m2 + m3) * l1 * l1;
    double a2 = i2 + m2 * r2 * r2 + m3 * l2 * l2;
    double a3 = i3 + m3 * r3 * r3;
    d.len[0] = (T)l1;
    d.len[1] = (T)l2;
    d.len[2] = (T)l3;
    d.a0_00 = (T)(a1 + a2 + a3);
    d.a0_01 = (T)(a2 + a3);
    d.a0_11 = (T)(a2 + a3);
    d.a3 = (T)a3;
    d.b12 = (T)((m2 * r2 + m3 * l2) * l1);
    d.b13 = (T)(m3 * r3 * l1);
    d.b23 = (T)(m3 * r3 * l2);
  }
  if (s.kind == CACTO_SYS_ALIENGO_LIPM) {
    d.omega = (T)s.p[0];
    d.sx = (T)s.p[1];
    d.sy = (T)s.p[2];
    d.delta0 = (T)s.p[3];
  }
  return d;
}

template <typename T>
CostDev<T> cost_dev(const cacto_cost_t& c) {
  CostDev<T> d{};
  d.kind = c.kind;
  d.n_obs = c.n_obstacles;
  d.tx = (T)c.target[0];
  d.ty = (T)c.target[1];
  for (int i = 0; i < CACTO_MAX_OBST; ++i) {
    d.ocx[i] = (T)c.obs_center[i][0];
    d.ocy[i] = (T)c.obs_center[i][1];
    d.e00[i] = (T)c.obs_form[i][0];
    d.e01[i] = (T)c.obs_form[i][1];
    d.e10[i] = (T)c.obs_form[i][2];
    d.e11[i] = (T)c.obs_form[i][3];
  }
  d.w_o = (T)c.w_obstacle;
  d.w_r = (T)c.w_reward;
  d.rho2 = (T)(c.reward_radius * c.reward_radius);
  d.inv_rho2 = (T)(1.0 / (c.reward_radius * c.reward_radius));
  d.w_u = (T)c.w_control;
  d.w_d = (T)c.w_distance;
  d.w_vel = (T)c.extra[0];
  d.w_vbar = (T)c.extra[1];
  d.v_max2 = (T)c.extra[2];
  d.obs_r2 = (T)c.extra[3];
  d.w_wall = (T)c.extra[4];
  return d;
}

template <int SYS> struct SysDims;
template <> struct SysDims<CACTO_SYS_TOY1D> { static constexpr int n = 1, m = 1; };
template <> struct SysDims<CACTO_SYS_POINTMASS> { static constexpr int n = 4, m = 2; };
template <> struct SysDims<CACTO_SYS_DUBINS> { static constexpr int n = 5, m = 2; };
template <> struct SysDims<CACTO_SYS_MANIPULATOR3> { static constexpr int n = 6, m = 3; };
template <> struct SysDims<CACTO_SYS_ALIENGO_LIPM> { static constexpr int n = 15, m = 6; };

// ---- manipulator rigid-body terms ------------------------------------------
// symmetric M(q) entries and the Coriolis vector h(q, dq), manipulator.py:51-84:
// h = sum_k dq_k dM_k dq - 0.5 [dq^T dM_i dq]_i  (c_ijk Christoffel identity)
template <typename T>
CACTO_D void manip_mass_trig(const SysDev<T>& P, const T* dq, T s2, T c2, T s3, T c3, T s23, T c23, T M[6],
                             T h[3]);
template <typename T>
CACTO_D void manip_mass(const SysDev<T>& P, const T* q, const T* dq, T M[6], T h[3]) {
  T s2, c2, s3, c3, s23, c23;
  m_sincos(q[1], &s2, &c2);
  m_sincos(q[2], &s3, &c3);
  m_sincos(q[1] + q[2], &s23, &c23);
  manip_mass_trig(P, dq, s2, c2, s3, c3, s23, c23, M, h);
}
template <typename T>
CACTO_D void manip_mass_trig(const SysDev<T>& P, const T* dq, T s2, T c2, T s3, T c3, T s23, T c23, T M[6],
                             T h[3]) {
  // M = A0 + c2 B12 + c23 B13 + c3 B23 -> (00, 01, 02, 11, 12, 22)
  M[0] = P.a0_00 + T(2) * P.b12 * c2 + T(2) * P.b13 * c23 + T(2) * P.b23 * c3;
  M[1] = P.a0_01 + P.b12 * c2 + P.b13 * c23 + T(2) * P.b23 * c3;
  M[2] = P.a3 + P.b13 * c23 + P.b23 * c3;
  M[3] = P.a0_11 + T(2) * P.b23 * c3;
  M[4] = P.a3 + P.b23 * c3;
  M[5] = P.a3;
  // dM_1 = -s2 B12 - s23 B13 ; dM_2 = -s23 B13 - s3 B23 (dM_0 = 0)
  T p12 = P.b12 * s2 + P.b13 * s23;
  T d1_00 = T(-2) * p12, d1_01 = -p12, d1_02 = -(P.b13 * s23);
  T t13 = P.b13 * s23, t23 = P.b23 * s3;
  T d2_00 = T(-2) * t13 - T(2) * t23, d2_01 = -t13 - T(2) * t23, d2_02 = -t13 - t23;
  T d2_11 = T(-2) * t23, d2_12 = -t23;
  // P1 = dM_1 dq, P2 = dM_2 dq
  T P1_0 = d1_00 * dq[0] + d1_01 * dq[1] + d1_02 * dq[2];
  T P1_1 = d1_01 * dq[0];
  T P1_2 = d1_02 * dq[0];
  T P2_0 = d2_00 * dq[0] + d2_01 * dq[1] + d2_02 * dq[2];
  T P2_1 = d2_01 * dq[0] + d2_11 * dq[1] + d2_12 * dq[2];
  T P2_2 = d2_02 * dq[0] + d2_12 * dq[1];
  T q1 = dq[0] * P1_0 + dq[1] * P1_1 + dq[2] * P1_2;
  T q2 = dq[0] * P2_0 + dq[1] * P2_1 + dq[2] * P2_2;
  h[0] = dq[1] * P1_0 + dq[2] * P2_0;
  h[1] = dq[1] * P1_1 + dq[2] * P2_1 - T(0.5) * q1;
  h[2] = dq[1] * P1_2 + dq[2] * P2_2 - T(0.5) * q2;
}

// inverse of the symmetric 3x3 (00, 01, 02, 11, 12, 22) -> same packing
template <typename T>
CACTO_D void sym3_inverse(const T M[6], T Mi[6]) {
  T c00 = M[3] * M[5] - M[4] * M[4];
  T c01 = M[2] * M[4] - M[1] * M[5];
  T c02 = M[1] * M[4] - M[2] * M[3];
  T det = M[0] * c00 + M[1] * c01 + M[2] * c02;
  T id;
  if constexpr (sizeof(T) == 4) id = __frcp_rn(det);  // == 1.f / det (IEEE rn), no division slow path
  else id = T(1) / det;
  Mi[0] = c00 * id;
  Mi[1] = c01 * id;
  Mi[2] = c02 * id;
  Mi[3] = (M[0] * M[5] - M[2] * M[2]) * id;
  Mi[4] = (M[1] * M[2] - M[0] * M[4]) * id;
  Mi[5] = (M[0] * M[3] - M[1] * M[1]) * id;
}

template <typename T>
CACTO_D void sym3_apply(const T A[6], const T* v, T* out) {
  out[0] = A[0] * v[0] + A[1] * v[1] + A[2] * v[2];
  out[1] = A[1] * v[0] + A[3] * v[1] + A[4] * v[2];
  out[2] = A[2] * v[0] + A[4] * v[1] + A[5] * v[2];
}

// ---- aliengo_lipm contact phase (oracle/aliengo.py) --------------------------
template <typename T>
struct LipmPhase {
  T ux, uy, ch, sh, gx, gy;
};
template <typename T>
CACTO_D LipmPhase<T> lipm_phase(const SysDev<T>& P, const T* x, const T* u) {
  LipmPhase<T> ph;
  T a = T(0.5) + u[4];
  T d = P.delta0 + u[5];
  T sig = m_cospi(x[8]);
  T sfx = P.sx, sfy = sig * P.sy, srx = -P.sx, sry = -sig * P.sy;
  // feet term + capture-point feedback cdot / omega (oracle/aliengo.py)
  ph.ux = a * (sfx - x[0]) + (T(1) - a) * (srx - x[2]) + x[6] / P.omega;
  ph.uy = a * (sfy - x[1]) + (T(1) - a) * (sry - x[3]) + x[7] / P.omega;
  ph.ch = m_cosh(P.omega * d);
  ph.sh = m_sinh(P.omega * d);
  ph.gx = (sfx - x[0]) - (srx - x[2]);
  ph.gy = (sfy - x[1]) - (sry - x[3]);
  return ph;
}

// rounded multiply / add that the compiler may not contract into an FMA: the
// Euler updates below then round exactly like NumPy's separate operations
CACTO_D float mul_rn(float a, float b) { return __fmul_rn(a, b); }
CACTO_D double mul_rn(double a, double b) { return __dmul_rn(a, b); }
CACTO_D float add_rn(float a, float b) { return __fadd_rn(a, b); }
CACTO_D double add_rn(double a, double b) { return __dadd_rn(a, b); }

// ---- x+ = f(x, u) --------------------------------------------------------------
template <int SYS, typename T>
CACTO_D void step(const SysDev<T>& P, const T* x, const T* u, T* xn) {
  const T dt = P.dt;
  if constexpr (SYS == CACTO_SYS_TOY1D) {
    xn[0] = add_rn(x[0], mul_rn(dt, u[0]));
  } else if constexpr (SYS == CACTO_SYS_POINTMASS) {
    xn[0] = add_rn(x[0], mul_rn(dt, x[2]));
    xn[1] = add_rn(x[1], mul_rn(dt, x[3]));
    xn[2] = add_rn(x[2], mul_rn(dt, u[0]));
    xn[3] = add_rn(x[3], mul_rn(dt, u[1]));
  } else if constexpr (SYS == CACTO_SYS_DUBINS) {
    T s, c;
    m_sincos(x[2], &s, &c);
    T dv = mul_rn(dt, x[3]);
    xn[0] = add_rn(x[0], mul_rn(dv, c));
    xn[1] = add_rn(x[1], mul_rn(dv, s));
    xn[2] = add_rn(x[2], mul_rn(dt, u[0]));
    xn[3] = add_rn(x[3], mul_rn(dt, x[4]));
    xn[4] = add_rn(x[4], mul_rn(dt, u[1]));
  } else if constexpr (SYS == CACTO_SYS_MANIPULATOR3) {
    T M[6], h[3], Mi[6], r[3], qdd[3];
    manip_mass(P, x, x + 3, M, h);
    sym3_inverse(M, Mi);
    r[0] = u[0] - h[0];
    r[1] = u[1] - h[1];
    r[2] = u[2] - h[2];
    sym3_apply(Mi, r, qdd);
    xn[0] = x[0] + dt * x[3];
    xn[1] = x[1] + dt * x[4];
    xn[2] = x[2] + dt * x[5];
    xn[3] = x[3] + dt * qdd[0];
    xn[4] = x[4] + dt * qdd[1];
    xn[5] = x[5] + dt * qdd[2];
  } else {  // aliengo_lipm
    LipmPhase<T> ph = lipm_phase(P, x, u);
    T sw = ph.sh / P.omega;
    xn[0] = u[0];
    xn[1] = u[1];
    xn[2] = u[2];
    xn[3] = u[3];
    xn[4] = x[4] + sw * x[6] + (T(1) - ph.ch) * ph.ux;
    xn[5] = x[5] + sw * x[7] + (T(1) - ph.ch) * ph.uy;
    xn[6] = ph.ch * x[6] - P.omega * ph.sh * ph.ux;
    xn[7] = ph.ch * x[7] - P.omega * ph.sh * ph.uy;
    xn[8] = x[8] + T(1);
#pragma unroll
    for (int i = 9; i < 15; ++i) xn[i] = x[i];
  }
}

// ---- f_u^T g (m-vector), the only Jacobian product the actor loss needs
// (nets.py:329); pointmass systems.py:50-54, dubins 82-94, manip 109-122 --------
template <int SYS, typename T>
CACTO_D void fu_t_g(const SysDev<T>& P, const T* x, const T* u, const T* g, T* out) {
  const T dt = P.dt;
  if constexpr (SYS == CACTO_SYS_TOY1D) {
    out[0] = dt * g[0];
  } else if constexpr (SYS == CACTO_SYS_POINTMASS) {
    out[0] = dt * g[2];
    out[1] = dt * g[3];
  } else if constexpr (SYS == CACTO_SYS_DUBINS) {
    out[0] = dt * g[2];
    out[1] = dt * g[4];
  } else if constexpr (SYS == CACTO_SYS_MANIPULATOR3) {
    T M[6], h[3], Mi[6], tmp[3];
    manip_mass(P, x, x + 3, M, h);
    sym3_inverse(M, Mi);
    sym3_apply(Mi, g + 3, tmp);  // (dt M^-1)^T g[3:6], M symmetric
    out[0] = dt * tmp[0];
    out[1] = dt * tmp[1];
    out[2] = dt * tmp[2];
  } else {
    LipmPhase<T> ph = lipm_phase(P, x, u);
    const T w = P.omega;
    out[0] = g[0];
    out[1] = g[1];
    out[2] = g[2];
    out[3] = g[3];
    out[4] = (T(1) - ph.ch) * (ph.gx * g[4] + ph.gy * g[5]) - w * ph.sh * (ph.gx * g[6] + ph.gy * g[7]);
    out[5] = (ph.ch * x[6] - w * ph.sh * ph.ux) * g[4] + (ph.ch * x[7] - w * ph.sh * ph.uy) * g[5] +
             (w * ph.sh * x[6] - w * w * ph.ch * ph.ux) * g[6] +
             (w * ph.sh * x[7] - w * w * ph.ch * ph.uy) * g[7];
  }
}

// ---- costs ------------------------------------------------------------------------
// reach / avoid field at the task point, costs.py:97-107
template <typename T>
CACTO_D T point_value(const CostDev<T>& C, T px, T py) {
  T rx = px - C.tx, ry = py - C.ty;
  T q = rx * rx + ry * ry;
  T val = C.w_d * q;
  // fp64 keeps NumPy's division (bit-level parity); fp32 multiplies by the
  // reciprocal (<= 1.5 ulp, as the input normalisation does)
  if constexpr (sizeof(T) == 4) val -= C.w_r * cost_exp(-q * C.inv_rho2);
  else val -= C.w_r * cost_exp(-q / C.rho2);
  // unrolled over the (uniform) obstacle count: no loop-carried index / constant-bank
  // address arithmetic per obstacle
#pragma unroll
  for (int i = 0; i < CACTO_MAX_OBST; ++i) {
    if (i >= C.n_obs) break;
    T dx = px - C.ocx[i], dy = py - C.ocy[i];
    T e = dx * (C.e00[i] * dx + C.e01[i] * dy) + dy * (C.e10[i] * dx + C.e11[i] * dy);
    val += C.w_o * cost_softplus(T(10) * (T(1) - e));
  }
  return val;
}

template <int SYS, typename T>
CACTO_D void task_point(const SysDev<T>& P, const T* x, T& px, T& py) {
  if constexpr (SYS == CACTO_SYS_MANIPULATOR3) {
    // manipulator.py:127-133: cumulative angles, summed link projections
    T a1 = x[0], a2 = x[0] + x[1], a3 = a2 + x[2];
    T s1, c1, s2, c2, s3, c3;
    m_sincos(a1, &s1, &c1);
    m_sincos(a2, &s2, &c2);
    m_sincos(a3, &s3, &c3);
    px = P.len[0] * c1 + P.len[1] * c2 + P.len[2] * c3;
    py = P.len[0] * s1 + P.len[1] * s2 + P.len[2] * s3;
  } else if constexpr (SYS == CACTO_SYS_ALIENGO_LIPM) {
    px = x[4];
    py = x[5];
  } else {
    px = x[0];
    py = SysDims<SYS>::n > 1 ? x[1] : T(0);
  }
}

// terminal cost l_T(x) (costs.py:78-79, 167-168; aliengo oracle/aliengo.py)
template <int SYS, typename T>
CACTO_D T terminal_cost(const SysDev<T>& P, const CostDev<T>& C, const T* x) {
  if constexpr (SYS == CACTO_SYS_TOY1D) {
    T s = x[0], w = s * s - T(1);
    return w * w + T(0.3) * s;
  } else if constexpr (SYS == CACTO_SYS_ALIENGO_LIPM) {
    T cx = x[4], cy = x[5], vx = x[6], vy = x[7];
    T q = cx * cx + cy * cy, v2 = vx * vx + vy * vy;
    T val = C.w_d * q;
    val -= C.w_r * cost_exp(-q / C.rho2);
    val += C.w_vel * v2;
    val += C.w_vbar * cost_softplus(T(10) * (v2 - C.v_max2));
    T ox = cx - x[9], oy = cy - x[10];
    val += C.w_o * cost_softplus(T(10) * (T(1) - (ox * ox + oy * oy) / C.obs_r2));
    val += C.w_wall * cost_softplus(T(10) * (x[11] - cx));
    val += C.w_wall * cost_softplus(T(10) * (cx - x[12]));
    val += C.w_wall * cost_softplus(T(10) * (x[13] - cy));
    val += C.w_wall * cost_softplus(T(10) * (cy - x[14]));
    return val;
  } else {
    T px, py;
    task_point<SYS>(P, x, px, py);
    return point_value(C, px, py);
  }
}

// stage cost l(x, u) then the Euler step x' = f(x, u) at the same x (the rollout
// and actor-loss epilogues).  fp32 manipulator: the six angle functions the two
// need (q2, q3, q2+q3 for M(q); q1, q1+q2, q1+q2+q3 for the end effector) come from
// three sincos and angle-addition products (the fp32 sums are rounded anyway);
// everything else (and fp64, for bit-level parity) calls the two separately.
template <int SYS, typename T>
CACTO_D T stage_cost(const SysDev<T>& P, const CostDev<T>& C, const T* x, const T* u);
template <int SYS, typename T>
CACTO_D T cost_and_step(const SysDev<T>& P, const CostDev<T>& C, bool has_cost, const T* x, const T* u, T* xn) {
  if constexpr (SYS == CACTO_SYS_MANIPULATOR3 && sizeof(T) == 4) {
    T s1, c1, s2, c2, s3, c3;
    m_sincos(x[0], &s1, &c1);
    m_sincos(x[1], &s2, &c2);
    m_sincos(x[2], &s3, &c3);
    const T s23 = s2 * c3 + c2 * s3, c23 = c2 * c3 - s2 * s3;
    T sc = T(0);
    if (has_cost) {
      const T s12 = s1 * c2 + c1 * s2, c12 = c1 * c2 - s1 * s2;
      const T s123 = s1 * c23 + c1 * s23, c123 = c1 * c23 - s1 * s23;
      const T px = P.len[0] * c1 + P.len[1] * c12 + P.len[2] * c123;
      const T py = P.len[0] * s1 + P.len[1] * s12 + P.len[2] * s123;
      T uu = u[0] * u[0];
      uu += u[1] * u[1];
      uu += u[2] * u[2];
      sc = point_value(C, px, py) + C.w_u * uu;
    }
    T M[6], h[3], Mi[6], r[3], qdd[3];
    manip_mass_trig(P, x + 3, s2, c2, s3, c3, s23, c23, M, h);
    sym3_inverse(M, Mi);
    r[0] = u[0] - h[0];
    r[1] = u[1] - h[1];
    r[2] = u[2] - h[2];
    sym3_apply(Mi, r, qdd);
    const T dt = P.dt;
    xn[0] = x[0] + dt * x[3];
    xn[1] = x[1] + dt * x[4];
    xn[2] = x[2] + dt * x[5];
    xn[3] = x[3] + dt * qdd[0];
    xn[4] = x[4] + dt * qdd[1];
    xn[5] = x[5] + dt * qdd[2];
    return sc;
  } else {
    const T sc = has_cost ? stage_cost<SYS>(P, C, x, u) : T(0);
    step<SYS>(P, x, u, xn);
    return sc;
  }
}

// stage cost l(x, u) = l_T(x) + w_u |u|^2 (costs.py:66-67, 147-149)
template <int SYS, typename T>
CACTO_D T stage_cost(const SysDev<T>& P, const CostDev<T>& C, const T* x, const T* u) {
  constexpr int m = SysDims<SYS>::m;
  T uu = u[0] * u[0];
#pragma unroll
  for (int j = 1; j < m; ++j) uu += u[j] * u[j];
  return terminal_cost<SYS>(P, C, x) + C.w_u * uu;
}

}  // namespace cacto
