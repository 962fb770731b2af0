// Pipelined parareal protocol of one time slice (host logic only, no CUDA):
// eq. parareal_correction, stopping rule eq. stop_criteria
// and the local exit of P:692-693 (retire when converged AND the
// predecessor retired; no global reduction).  The GPU driver (pif_parareal)
// and the CPU test export (pif_debug_parareal_protocol) run this same code
// with different operations.
#include <math.h>

#include <utility>

#include "pif_internal.cuh"

namespace pif {

pif_status run_pipeline(int t, int T, int max_iter, double tol, const ProtocolOps& ops,
                        ProtocolResult& res) {
  int U = PB_U, Fk = PB_F, Gold = PB_GOLD, Gnew = PB_GNEW, Unext = PB_UNEXT;
  res.iterations = 0;
  res.retired_at = -1;
  res.ex.assign(max_iter, NAN);
  res.ev.assign(max_iter, NAN);
  res.final_buf = Gold;  // U_{t+1}^0 if no correction iteration runs
  bool pred_retired = (t == 0), retired = false;
  pif_status s;
  double flag = 0.0;
  // iteration 0: U_t^0 from the predecessor's coarse sweep, U_{t+1}^0 = G(U_t^0)
  s = (t == 0) ? ops.store_initial(ops.user, U) : ops.recv(ops.user, U, &flag);
  if (s != PIF_OK) return s;
  if ((s = ops.propagate(ops.user, 1, U, Gold)) != PIF_OK) return s;
  if (t + 1 < T && (s = ops.send(ops.user, Gold, 0.0)) != PIF_OK) return s;
  bool changed = false;  // U_t changed since Gold = G(U_t) was computed
  for (int k = 0; k < max_iter && !retired; ++k) {
    res.iterations = k + 1;
    if ((s = ops.propagate(ops.user, 0, U, Fk)) != PIF_OK) return s;  // F(U_t^k)
    if (!pred_retired) {                                                // U_t^{k+1}
      if ((s = ops.recv(ops.user, U, &flag)) != PIF_OK) return s;
      if (flag != 0.0) pred_retired = true;
      changed = true;
    }
    if ((s = ops.guard(ops.user)) != PIF_OK) return s;
    int Gn = Gold;  // an unchanged input gives G(U_t^{k+1}) = G(U_t^k) exactly
    if (changed) {
      if ((s = ops.propagate(ops.user, 1, U, Gnew)) != PIF_OK) return s;
      Gn = Gnew;
    }
    double ex = 0.0, ev = 0.0;
    if ((s = ops.correct(ops.user, Fk, Gn, Gold, Unext, &ex, &ev)) != PIF_OK) return s;
    changed = false;
    if (Gn == Gnew) std::swap(Gold, Gnew);
    res.ex[k] = ex;
    res.ev[k] = ev;
    res.final_buf = Unext;
    if (ex <= tol && ev <= tol && pred_retired) {
      retired = true;
      res.retired_at = k + 1;
    }
    if (t + 1 < T && (s = ops.send(ops.user, Unext, retired ? 1.0 : 0.0)) != PIF_OK) return s;
  }
  return PIF_OK;
}

}  // namespace pif

// ----------------------------------------------------- test-only export --
namespace {
struct CallbackOps {
  const pif_protocol_ops* o;
};
pif_status cb_store(void* u, int dst) {
  auto* o = static_cast<CallbackOps*>(u)->o;
  return (pif_status)o->store_initial(o->user, dst);
}
pif_status cb_prop(void* u, int which, int src, int dst) {
  auto* o = static_cast<CallbackOps*>(u)->o;
  return (pif_status)o->propagate(o->user, which, src, dst);
}
pif_status cb_correct(void* u, int f, int gn, int go, int un, double* ex, double* ev) {
  auto* o = static_cast<CallbackOps*>(u)->o;
  return (pif_status)o->correct(o->user, f, gn, go, un, ex, ev);
}
pif_status cb_send(void* u, int buf, double flag) {
  auto* o = static_cast<CallbackOps*>(u)->o;
  return (pif_status)o->send(o->user, buf, flag);
}
pif_status cb_recv(void* u, int buf, double* flag) {
  auto* o = static_cast<CallbackOps*>(u)->o;
  return (pif_status)o->recv(o->user, buf, flag);
}
pif_status cb_guard(void*) { return PIF_OK; }
}  // namespace

extern "C" pif_status pif_debug_parareal_protocol(int32_t t, int32_t T, int32_t max_iter,
                                                  double tol, const pif_protocol_ops* ops,
                                                  int32_t* iterations, int32_t* retired_at,
                                                  double* err_x, double* err_v,
                                                  int32_t* final_buf) {
  if (!ops || !iterations || !retired_at || !err_x || !err_v || !final_buf || T < 1 || t < 0 ||
      t >= T || max_iter < 0)
    return PIF_ERR_ARG;
  CallbackOps cb{ops};
  pif::ProtocolOps po{&cb, cb_store, cb_prop, cb_correct, cb_send, cb_recv, cb_guard};
  pif::ProtocolResult res;
  pif_status s = pif::run_pipeline(t, T, max_iter, tol, po, res);
  if (s != PIF_OK) return s;
  *iterations = res.iterations;
  *retired_at = res.retired_at;
  for (int k = 0; k < max_iter; ++k) {
    err_x[k] = res.ex[k];
    err_v[k] = res.ev[k];
  }
  *final_buf = res.final_buf;
  return PIF_OK;
}
