"""Minimax coefficients of the table exp's polynomial (gs_device.cuh, GS_EXP_TBL_BITS = 7).

e1(u) = u (C1 + C2 u + ... + C_deg u^(deg-1)) approximates e^(u ln2 / T) - 1 on |u| <= 1/2 with the
smallest maximum absolute error (Remez exchange in 60-digit arithmetic); the table exp returns
T[k] (1 + e1(u)), so that error is the relative error of G beyond the table's rounding.

    python tools/exp_minimax.py      # T = 128, degree 4: max error 7.6e-17 (64 / degree-5 Taylor: 3.5e-17)
"""
import mpmath as mp
mp.mp.dps = 60
def remez(T, deg, iters=30):
    # e1(u) = u * P(u), P degree deg-1; minimize max |u P(u) - (exp(u ln2/T) - 1)| on [-1/2, 1/2]
    a = mp.log(2)/T
    f = lambda u: mp.expm1(u*a)
    m = deg  # unknowns c1..c_deg plus E
    # initial reference: Chebyshev extrema, deg+1 points
    pts = [mp.mpf(0.5)*mp.cos(mp.pi*k/deg) for k in range(deg+1)]
    for it in range(iters):
        A = mp.matrix(deg+1, deg+1); b = mp.matrix(deg+1, 1)
        for i,u in enumerate(pts):
            for j in range(deg): A[i,j] = u**(j+1)
            A[i,deg] = (-1)**i
            b[i] = f(u)
        sol = mp.lu_solve(A, b)
        c = [sol[j] for j in range(deg)]
        err = lambda u: sum(c[j]*u**(j+1) for j in range(deg)) - f(u)
        # find extrema on a fine grid then refine
        N = 4000
        grid = [mp.mpf(-0.5) + mp.mpf(k)/N for k in range(N+1)]
        vals = [err(u) for u in grid]
        ext = [0]
        for k in range(1, N):
            if (vals[k]-vals[k-1])*(vals[k+1]-vals[k]) <= 0: ext.append(k)
        ext.append(N)
        ext = [grid[k] for k in ext]
        if len(ext) != deg+1:
            # keep alternating subset of largest
            pass
        pts = ext[:deg+1] if len(ext) >= deg+1 else pts
    E = max(abs(err(u)) for u in grid)
    return c, E
for T, deg in [(128, 4), (256, 4)]:
    c, E = remez(T, deg)
    taylor = (mp.log(2)/T/2)**(deg+1)/mp.factorial(deg+1)
    print(T, deg, "minimax err %.3e" % float(E), "taylor trunc %.3e" % float(taylor))
    print("  ", [mp.nstr(x, 20) for x in c])
    print("  as double:", [repr(float(x)) for x in c])
