// control.cpp -- host LAPACK shim for the cycle-end control work: the
// generalised eigenproblem of order k+s (finalGenEigValue)
// and the k x k SVD (equationSVD).
//
// There is no system LAPACK in this image; the library dlopen()s the OpenBLAS
// that scipy ships (symbols prefixed `scipy_`), whose path the Python binding
// exports as $RBICG_LAPACK.  Plain (unprefixed) names are tried as fallback.
#include <dlfcn.h>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace rbicg {

typedef void (*dggev_t)(const char *, const char *, const int *, double *, const int *, double *,
                        const int *, double *, double *, double *, double *, const int *, double *,
                        const int *, double *, const int *, int *, size_t, size_t);
typedef void (*zggev_t)(const char *, const char *, const int *, cplx *, const int *, cplx *,
                        const int *, cplx *, cplx *, cplx *, const int *, cplx *, const int *,
                        cplx *, const int *, double *, int *, size_t, size_t);
typedef void (*dgesvd_t)(const char *, const char *, const int *, const int *, double *,
                         const int *, double *, double *, const int *, double *, const int *,
                         double *, const int *, int *, size_t, size_t);
typedef void (*zgesvd_t)(const char *, const char *, const int *, const int *, cplx *, const int *,
                         double *, cplx *, const int *, cplx *, const int *, cplx *, const int *,
                         double *, int *, size_t, size_t);

typedef void (*dgeev_t)(const char *, const char *, const int *, double *, const int *, double *,
                        double *, double *, const int *, double *, const int *, double *,
                        const int *, int *, size_t, size_t);
typedef void (*zgeev_t)(const char *, const char *, const int *, cplx *, const int *, cplx *,
                        cplx *, const int *, cplx *, const int *, cplx *, const int *, double *,
                        int *, size_t, size_t);

static struct {
  std::once_flag once;
  void *h = nullptr;
  dgeev_t dgeev = nullptr;
  zgeev_t zgeev = nullptr;
  dggev_t dggev = nullptr;
  zggev_t zggev = nullptr;
  dgesvd_t dgesvd = nullptr;
  zgesvd_t zgesvd = nullptr;
  int (*set_threads_local)(int) = nullptr;   // OpenBLAS >= 0.3.27, per calling thread
} L;

static void *sym(const char *name) {
  std::string a = std::string("scipy_") + name;
  void *p = dlsym(L.h, a.c_str());
  if (!p) p = dlsym(L.h, name);
  return p;
}

static void load() {
  std::call_once(L.once, [] {
    const char *path = getenv("RBICG_LAPACK");
    if (path) L.h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!L.h) L.h = dlopen("liblapack.so.3", RTLD_NOW | RTLD_LOCAL);
    if (!L.h) L.h = dlopen("libopenblas.so.0", RTLD_NOW | RTLD_LOCAL);
    if (!L.h) return;
    L.dgeev = (dgeev_t)sym("dgeev_");
    L.zgeev = (zgeev_t)sym("zgeev_");
    L.dggev = (dggev_t)sym("dggev_");
    L.zggev = (zggev_t)sym("zggev_");
    L.dgesvd = (dgesvd_t)sym("dgesvd_");
    L.zgesvd = (zgesvd_t)sym("zgesvd_");
    L.set_threads_local = (int (*)(int))dlsym(L.h, "openblas_set_num_threads_local");
  });
  RB_CHECK(L.dggev && L.zggev && L.dgesvd && L.zgesvd && L.dgeev && L.zgeev, RBICG_ELAPACK);
  // The pencils are of order <= k + s (<= 70): OpenBLAS's thread pool costs
  // more than it saves there (C3 general-case cycle end: ~10 ms of host eig
  // per cycle with the default pool) -- one thread for this calling thread
  if (L.set_threads_local) L.set_threads_local(1);
}

// Standard eigenproblem P w = λ w with left and right vectors (the Q = I
// pencil of the first cycle of the first system, eigenvectors of T_1,
// P:614-628): the QR algorithm instead of QZ, same outputs as lapack_ggev
// with beta = 1.
int lapack_geev(bool real, int m, const std::vector<cplx> &P, std::vector<cplx> &alpha,
                std::vector<cplx> &beta, std::vector<cplx> &VL, std::vector<cplx> &VR) {
  load();
  alpha.assign(m, 0.0);
  beta.assign(m, 1.0);
  VL.assign((size_t)m * m, 0.0);
  VR.assign((size_t)m * m, 0.0);
  if (m == 0) return 0;
  int info = 0;
  const char V = 'V';
  if (real) {
    std::vector<double> a((size_t)m * m), vl((size_t)m * m), vr((size_t)m * m), wr(m), wi(m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) a[(size_t)j * m + i] = P[(size_t)i * m + j].real();
    int lwork = -1;
    double wq = 0;
    L.dgeev(&V, &V, &m, a.data(), &m, wr.data(), wi.data(), vl.data(), &m, vr.data(), &m, &wq, &lwork,
            &info, 1, 1);
    lwork = std::max(1, (int)wq);
    std::vector<double> work(lwork);
    L.dgeev(&V, &V, &m, a.data(), &m, wr.data(), wi.data(), vl.data(), &m, vr.data(), &m,
            work.data(), &lwork, &info, 1, 1);
    if (info != 0) return RBICG_ELAPACK;
    for (int j = 0; j < m; ++j) alpha[j] = cplx(wr[j], wi[j]);
    for (int j = 0; j < m; ++j) {
      if (wi[j] == 0.0) {
        for (int i = 0; i < m; ++i) {
          VR[(size_t)j * m + i] = vr[(size_t)j * m + i];
          VL[(size_t)j * m + i] = vl[(size_t)j * m + i];
        }
      } else if (wi[j] > 0.0 && j + 1 < m) {   // conjugate pair in adjacent columns
        for (int i = 0; i < m; ++i) {
          const cplx cr(vr[(size_t)j * m + i], vr[(size_t)(j + 1) * m + i]);
          const cplx cl(vl[(size_t)j * m + i], vl[(size_t)(j + 1) * m + i]);
          VR[(size_t)j * m + i] = cr;
          VR[(size_t)(j + 1) * m + i] = std::conj(cr);
          VL[(size_t)j * m + i] = cl;
          VL[(size_t)(j + 1) * m + i] = std::conj(cl);
        }
        ++j;
      }
    }
  } else {
    std::vector<cplx> a((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) a[(size_t)j * m + i] = P[(size_t)i * m + j];
    int lwork = -1;
    cplx wq;
    std::vector<double> rwork(2 * m);
    L.zgeev(&V, &V, &m, a.data(), &m, alpha.data(), VL.data(), &m, VR.data(), &m, &wq, &lwork,
            rwork.data(), &info, 1, 1);
    lwork = std::max(1, (int)wq.real());
    std::vector<cplx> work(lwork);
    L.zgeev(&V, &V, &m, a.data(), &m, alpha.data(), VL.data(), &m, VR.data(), &m, work.data(),
            &lwork, rwork.data(), &info, 1, 1);
    if (info != 0) return RBICG_ELAPACK;
  }
  return 0;
}

// P, Q row-major m x m.  Outputs: alpha, beta (complex), VL, VR column-major
// m x m complex (column j = eigenvector of pair j).  pair_first unused (the
// conjugate partner of a complex pair of a real pencil is the adjacent index).
int lapack_ggev(bool real, int m, std::vector<cplx> P, std::vector<cplx> Q,
                std::vector<cplx> &alpha, std::vector<cplx> &beta, std::vector<cplx> &VL,
                std::vector<cplx> &VR, std::vector<int> &pair_first) {
  load();
  alpha.assign(m, 0.0);
  beta.assign(m, 0.0);
  VL.assign((size_t)m * m, 0.0);
  VR.assign((size_t)m * m, 0.0);
  pair_first.assign(m, -1);
  if (m == 0) return 0;
  int info = 0;
  const char V = 'V';
  if (real) {
    std::vector<double> a((size_t)m * m), b((size_t)m * m), vl((size_t)m * m), vr((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        a[(size_t)j * m + i] = P[(size_t)i * m + j].real();
        b[(size_t)j * m + i] = Q[(size_t)i * m + j].real();
      }
    std::vector<double> ar(m), ai(m), be(m);
    int lwork = -1;
    double wq = 0;
    L.dggev(&V, &V, &m, a.data(), &m, b.data(), &m, ar.data(), ai.data(), be.data(), vl.data(),
            &m, vr.data(), &m, &wq, &lwork, &info, 1, 1);
    lwork = std::max(1, (int)wq);
    std::vector<double> work(lwork);
    L.dggev(&V, &V, &m, a.data(), &m, b.data(), &m, ar.data(), ai.data(), be.data(), vl.data(),
            &m, vr.data(), &m, work.data(), &lwork, &info, 1, 1);
    if (info != 0) return RBICG_ELAPACK;
    for (int j = 0; j < m; ++j) {
      alpha[j] = cplx(ar[j], ai[j]);
      beta[j] = cplx(be[j], 0.0);
    }
    for (int j = 0; j < m; ++j) {
      if (ai[j] == 0.0) {
        for (int i = 0; i < m; ++i) {
          VR[(size_t)j * m + i] = vr[(size_t)j * m + i];
          VL[(size_t)j * m + i] = vl[(size_t)j * m + i];
        }
      } else if (ai[j] > 0.0 && j + 1 < m) {
        for (int i = 0; i < m; ++i) {
          const cplx wr(vr[(size_t)j * m + i], vr[(size_t)(j + 1) * m + i]);
          const cplx wl(vl[(size_t)j * m + i], vl[(size_t)(j + 1) * m + i]);
          VR[(size_t)j * m + i] = wr;
          VR[(size_t)(j + 1) * m + i] = std::conj(wr);
          VL[(size_t)j * m + i] = wl;
          VL[(size_t)(j + 1) * m + i] = std::conj(wl);
        }
        pair_first[j] = j;
        pair_first[j + 1] = j;
        ++j;
      }
    }
  } else {
    std::vector<cplx> a((size_t)m * m), b((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        a[(size_t)j * m + i] = P[(size_t)i * m + j];
        b[(size_t)j * m + i] = Q[(size_t)i * m + j];
      }
    int lwork = -1;
    cplx wq;
    std::vector<double> rwork(8 * m);
    L.zggev(&V, &V, &m, a.data(), &m, b.data(), &m, alpha.data(), beta.data(), VL.data(), &m,
            VR.data(), &m, &wq, &lwork, rwork.data(), &info, 1, 1);
    lwork = std::max(1, (int)wq.real());
    std::vector<cplx> work(lwork);
    L.zggev(&V, &V, &m, a.data(), &m, b.data(), &m, alpha.data(), beta.data(), VL.data(), &m,
            VR.data(), &m, work.data(), &lwork, rwork.data(), &info, 1, 1);
    if (info != 0) return RBICG_ELAPACK;
  }
  return 0;
}

// G row-major m x m.  G = Mleft diag(S) Nright^H; Mleft, Nright column-major.
int lapack_gesvd(bool real, int m, std::vector<cplx> G, std::vector<double> &S,
                 std::vector<cplx> &Mleft, std::vector<cplx> &Nright) {
  load();
  S.assign(m, 0.0);
  Mleft.assign((size_t)m * m, 0.0);
  Nright.assign((size_t)m * m, 0.0);
  if (m == 0) return 0;
  int info = 0;
  const char A = 'A';
  if (real) {
    std::vector<double> a((size_t)m * m), u((size_t)m * m), vt((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) a[(size_t)j * m + i] = G[(size_t)i * m + j].real();
    int lwork = -1;
    double wq = 0;
    L.dgesvd(&A, &A, &m, &m, a.data(), &m, S.data(), u.data(), &m, vt.data(), &m, &wq, &lwork,
             &info, 1, 1);
    lwork = std::max(1, (int)wq);
    std::vector<double> work(lwork);
    L.dgesvd(&A, &A, &m, &m, a.data(), &m, S.data(), u.data(), &m, vt.data(), &m, work.data(),
             &lwork, &info, 1, 1);
    if (info != 0) return RBICG_ELAPACK;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        Mleft[(size_t)j * m + i] = u[(size_t)j * m + i];
        Nright[(size_t)j * m + i] = vt[(size_t)i * m + j];   // N = VT^T
      }
  } else {
    std::vector<cplx> a((size_t)m * m), u((size_t)m * m), vt((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) a[(size_t)j * m + i] = G[(size_t)i * m + j];
    int lwork = -1;
    cplx wq;
    std::vector<double> rwork(5 * m + 8);
    L.zgesvd(&A, &A, &m, &m, a.data(), &m, S.data(), u.data(), &m, vt.data(), &m, &wq, &lwork,
             rwork.data(), &info, 1, 1);
    lwork = std::max(1, (int)wq.real());
    std::vector<cplx> work(lwork);
    L.zgesvd(&A, &A, &m, &m, a.data(), &m, S.data(), u.data(), &m, vt.data(), &m, work.data(),
             &lwork, rwork.data(), &info, 1, 1);
    if (info != 0) return RBICG_ELAPACK;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        Mleft[(size_t)j * m + i] = u[(size_t)j * m + i];
        Nright[(size_t)j * m + i] = std::conj(vt[(size_t)i * m + j]);   // N = VT^H
      }
  }
  return 0;
}

}  // namespace rbicg
