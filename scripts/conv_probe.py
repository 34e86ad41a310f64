"""a3/a4 alternatives, measured: the grid
convolution phi(a) = sum_b K(delta (a - b)) q(b) on an N x N node lattice
(spacing delta = h/3), done three ways on the GPU at the grid sizes of the
bench windows (N = 60 .. 162):

  fft     libtsnet's own chain (k_row_fwd + k_col + k_row_inv: kernel
          tabulation, forward FFTs, Parseval Z, 6 products, inverse FFTs),
          timed as one captured tsnet_grad_parts on a small P (n = 1024, so
          the spread and SpMV are a few us) -- an upper bound of the chain;
  sep     separable low rank: T[mx, my] = K(delta mx, delta my) on the
          (2N-1)^2 offsets, SVD (cuSOLVER, fp64) truncated at sigma_r <
          1e-7 sigma_1, then phi = sum_r U_r Q V_r^T with Toeplitz U_r, V_r
          (batched cuBLAS GEMM: fp64 = DMMA tensor cores, fp32 = SGEMM);
          the SVD must be redone every iteration (delta follows the bbox);
  dense   the direct N^2 x N^2 Toeplitz-block matrix times the charges (fp32
          SGEMM and fp64), its matrix built every iteration.

Kernels: K1 = 1/(1+r^2), K2 = K1^2, Ke = 1/(eps+r^2), and the offset forms
dx K2, dy K2, dx Ke, dy Ke (7 kernels) against 3 charge channels (W1, Mx, My)
as the local-moment field needs.  Library GEMM/SVD/FFT here are a
probe, not the product.  Accuracy: relL2 against an fp64 FFT of the same
convolution.

    python scripts/conv_probe.py [N ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

dev = torch.device("cuda")
EPS = 0.05


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, out   # us


def kernels(dx, dy):
    r2 = dx * dx + dy * dy
    k1 = 1.0 / (1.0 + r2)
    k2 = k1 * k1
    ke = 1.0 / (EPS + r2)
    return [k1, k2, ke, dx * k2, dy * k2, dx * ke, dy * ke]


def reference(T, Q, N):
    """fp64 FFT convolution: out[k, c] = sum_b T_k[a - b] Q_c[b] (linear)."""
    M = 2 * N
    Tf = torch.fft.rfft2(torch.roll(torch.nn.functional.pad(T, (0, 1, 0, 1)), shifts=(-(N - 1), -(N - 1)),
                                    dims=(-2, -1)), s=(M, M))
    Qf = torch.fft.rfft2(Q, s=(M, M))
    out = torch.fft.irfft2(Tf[:, None] * Qf[None], s=(M, M))
    return out[..., :N, :N]


def toeplitz(u, N):
    """(R, 2N-1) -> (R, N, N), X[a, b] = u[a - b + N - 1]."""
    idx = (torch.arange(N, device=u.device)[:, None] - torch.arange(N, device=u.device)[None, :]) + N - 1
    return u[:, idx]


def probe_sep(T, Q, N, dtype):
    def run():
        outs = []
        for k in range(T.shape[0]):
            U, S, Vh = torch.linalg.svd(T[k])
            R = int((S > 1e-7 * S[0]).sum().item())
            s = S[:R].sqrt()
            X = toeplitz((U[:, :R] * s).T.contiguous(), N).to(dtype)      # (R, N, N)
            Yt = toeplitz((Vh[:R].T * s).T.contiguous(), N).to(dtype)     # (R, N, N)
            Z = torch.matmul(X[:, None], Q.to(dtype)[None])               # (R, 3, N, N)
            Z = torch.matmul(Z, Yt[:, None].transpose(-1, -2))
            outs.append(Z.sum(0))
        return torch.stack(outs), R
    return run


def probe_dense(T, Q, N, dtype):
    ii = torch.arange(N, device=dev)
    da = (ii[:, None] - ii[None, :]) + N - 1                              # (N, N)

    def run():
        outs = []
        for k in range(T.shape[0]):
            # K[(a1, a2), (b1, b2)] = T[a1 - b1, a2 - b2]
            Km = T[k][da[:, None, :, None], da[None, :, None, :]].reshape(N * N, N * N).to(dtype)
            outs.append((Km @ Q.to(dtype).reshape(3, N * N).T).T.reshape(3, N, N))
        return torch.stack(outs)
    return run


def probe_fft_chain(N):
    from paper_2509_19785_b200 import GradParams, alloc_workspace, tsnet_build_P, tsnet_grad_parts, tsnet_read_stats
    from workloads import config_graph, uniform_layout
    ip, ix = config_graph(1)
    P = tsnet_build_P(torch.from_numpy(ip).to(dev), torch.from_numpy(ix).to(dev), u=40.0, seed=0)["P"]
    S = (N // 3) * 0.25 - 0.01
    Y = torch.from_numpy(uniform_layout(P.n, S, 1)).to(dev)
    gp = GradParams(1.0, 0.01, 0.6)
    ws = alloc_workspace(P.n, P.nnz, gp, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        tsnet_grad_parts(P, Y, gp, ws, stream=s)
        s.synchronize()
        st = tsnet_read_stats(ws, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tsnet_grad_parts(P, Y, gp, ws, stream=s)
    torch.cuda.synchronize()
    us, _ = timed(lambda: g.replay(), 50)
    return us, st["N"]


def main():
    Ns = [int(a) for a in sys.argv[1:]] or [60, 108, 162]
    torch.manual_seed(0)
    for N in Ns:
        h = 0.25
        delta = h / 3
        m = torch.arange(-(N - 1), N, device=dev, dtype=torch.float64) * delta
        T = torch.stack(kernels(m[:, None], m[None, :]))                 # (7, 2N-1, 2N-1)
        Q = torch.rand(3, N, N, device=dev, dtype=torch.float64)
        ref = reference(T, Q, N)
        row = {"N": N}
        try:
            us, Ngot = probe_fft_chain(N)
            row["fft_chain_us"] = round(us, 2)
            row["fft_chain_N"] = Ngot
        except Exception as e:   # noqa: BLE001
            row["fft_chain_error"] = str(e)[:200]
        for name, dt in (("sep_fp64", torch.float64), ("sep_fp32", torch.float32)):
            us, (out, R) = timed(probe_sep(T, Q, N, dt), 5)
            row[name + "_us"] = round(us, 1)
            row[name + "_rank_last_kernel"] = R
            row[name + "_relL2"] = float((out.double() - ref).norm() / ref.norm())
        if N <= 108:
            for name, dt in (("dense_fp64", torch.float64), ("dense_fp32", torch.float32)):
                us, out = timed(probe_dense(T, Q, N, dt), 5)
                row[name + "_us"] = round(us, 1)
                row[name + "_relL2"] = float((out.double() - ref).norm() / ref.norm())
        # the GEMM part of the separable form alone (rank 16, factors given)
        R = 16
        for name, dt in (("sep_gemm_only_fp64", torch.float64), ("sep_gemm_only_fp32", torch.float32)):
            X = torch.rand(7 * R, 1, N, N, device=dev, dtype=dt)
            Qd = Q.to(dt)[None]

            def g():
                return torch.matmul(torch.matmul(X, Qd), X.transpose(-1, -2))
            us, _ = timed(g, 20)
            row[name + "_us"] = round(us, 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
