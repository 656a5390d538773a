"""Shared-memory bank-conflict model of the generic element kernel's 3D
sweeps (tmop_elem.cuh f1/f2/f3, b3/b2/b1) for one element per CTA (EPB = 1):
extra 64-bit wavefronts per element, searched over the strides of the U / Bv
buffer [c][v][qz][ky][kx] (UZ, UV, UC) and of the W / A buffer
[c][v3][qz][qy][kx] (WY, WZ, WV, WC).  The U and W buffers are accessed by
disjoint stage pairs (f1/f2 + b2/b1 and f2/f3 + b3/b2), so they are searched
independently.  Prints the chosen strides for tmop_elem.cuh's ElemPad.
    python tools/elem_banks.py 5 6 128"""
import itertools
import sys

from xl_banks import ideal, waves


def _stage(items, NT, addr, js):
    tot = 0
    for j in js:
        for base in range(0, items, NT):
            for w0 in range(base, base + NT, 32):
                a = [addr(w, j) if w < items else None for w in range(w0, w0 + 32)]
                tot += waves(a) - ideal(a)
    return tot


def u_extra(N, Q, NT, UZ, UV, UC, C=3):
    NN, QN = N * N, Q * N
    t = 0
    for v in (0, 1):   # f1 write U / b1 read Bv: item (c, ky, kx), j = qz
        t += _stage(C * NN, NT, lambda w, q: (w // NN) * UC + v * UV + q * UZ + w % NN, range(Q))
    for v in (0, 1):   # f2 read U / b2 write Bv: item (c, qz, kx), j = ky
        t += _stage(C * QN, NT, lambda w, k: (w // QN) * UC + v * UV + ((w % QN) // N) * UZ + k * N + w % N, range(N))
    return 2 * t


def w_extra(N, Q, NT, WY, WZ, WV, WC, C=3):
    QN, QQ = Q * N, Q * Q
    t = 0
    for v in (0, 1, 2):   # f2 write W / b2 read A: item (c, qz, kx), j = qy
        t += _stage(C * QN, NT, lambda w, q: (w // QN) * WC + v * WV + ((w % QN) // N) * WZ + q * WY + w % N, range(Q))
    for v in (0, 1, 2):   # f3 read W / b3 write A: item (c, qz, qy), j = kx
        t += _stage(C * QQ, NT, lambda w, k: (w // QQ) * WC + v * WV + ((w % QQ) // Q) * WZ + (w % Q) * WY + k, range(N))
    return 2 * t


def search(N, Q, NT):
    NN = N * N
    cur_u = u_extra(N, Q, NT, NN, Q * NN, 2 * Q * NN)
    ub = min((u_extra(N, Q, NT, UZ, UV, UC), UC - 2 * Q * NN, UZ, UV, UC)
             for UZ in range(NN, NN + 16) for UV in range(Q * UZ, Q * UZ + 16, 1)
             for UC in range(2 * UV, 2 * UV + 16, 1))
    WY0 = N | 1
    cur_w = w_extra(N, Q, NT, WY0, Q * WY0, Q * Q * WY0, 3 * Q * Q * WY0)
    wb = min((w_extra(N, Q, NT, WY, WZ, WV, WC), WC - 3 * Q * Q * N, WY, WZ, WV, WC)
             for WY in range(N, N + 3) for WZ in range(Q * WY, Q * WY + 16)
             for WV in range(Q * WZ, Q * WZ + 16, 2) for WC in range(3 * WV, 3 * WV + 16, 2))
    return cur_u, ub, cur_w, wb


if __name__ == "__main__":
    N, Q, NT = (int(s) for s in sys.argv[1:4])
    cu, ub, cw, wb = search(N, Q, NT)
    print(f"N={N} Q={Q} NT={NT}: U extra {cu} -> {ub[0]} (UZ {ub[2]} UV {ub[3]} UC {ub[4]}); "
          f"W extra {cw} -> {wb[0]} (WY {wb[2]} WZ {wb[3]} WV {wb[4]} WC {wb[5]})")
