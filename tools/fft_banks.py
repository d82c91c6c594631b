"""Shared-memory bank-conflict model of the register FFT passes (fft_reg.cuh):
for each N and candidate layout, the mean number of 128-byte wavefronts per
warp-wide float2 access (ideal 2.0) over every pass's loads/stores and the
digit-reversed output read.  Not part of the product."""
import itertools
PLANS = {64: [16, 4], 128: [16, 8], 256: [16, 16], 512: [16, 16, 2], 1024: [16, 16, 4],
         2048: [16, 16, 8], 4096: [16, 16, 16]}

def wavefronts(addrs):           # addrs: float2 element indices of 32 lanes
    n = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(half):
            banks.setdefault(a % 16, set()).add(a)
        n += max(len(v) for v in banks.values())
    return n

def out_pos(N, k):
    pos, M, rem = 0, N, k
    for R in PLANS[N]:
        M //= R; pos += (rem % R) * M; rem //= R
    return pos

def score(N, lay):
    T = N // 16; tot = cnt = 0
    M = N
    for R in PLANS[N]:
        Mp = M // R
        for q in range(16 // R):
            for w0 in range(0, T, 32):
                lanes = [w0 + l for l in range(32) if w0 + l < T]
                if len(lanes) < 32: lanes = lanes + lanes[: 32 - len(lanes)]
                for n1 in range(R):
                    addrs = []
                    for tt in lanes:
                        item = tt + q * T; g, n2 = divmod(item, Mp)
                        addrs.append(lay(g * M + n2 + n1 * Mp))
                    tot += wavefronts(addrs); cnt += 1
        M = Mp
    ro = 0; rc = 0
    for k0 in range(0, N, 32):
        ro += wavefronts([lay(out_pos(N, k0 + l)) for l in range(32)]); rc += 1
    return tot / cnt, ro / rc

cands = {
    "pad32 (i + i>>5)": lambda e: e + (e >> 5),
    "pad16 (i + i>>4)": lambda e: e + (e >> 4),
    "pad16+pad256": lambda e: e + (e >> 4) + (e >> 8),
    "xor (i ^ (i>>4)&15)": lambda e: e ^ ((e >> 4) & 15),
    "xor2 (i ^ ((i>>4)^(i>>8))&15)": lambda e: e ^ (((e >> 4) ^ (e >> 8)) & 15),
    "xor3 (i ^ ((i>>4)+(i>>8)*?)&15)": lambda e: e ^ (((e >> 4) + 5 * (e >> 8)) & 15),
}
for name, lay in cands.items():
    print(f"{name:34s}", "  ".join(f"N={N}: pass {a:.2f} out {b:.2f}" for N, (a, b) in
                                   ((N, score(N, lay)) for N in (256, 512, 1024, 2048, 4096))))
