"""Fig. 1 of the paper: split width alpha of the four convolution variants in
single precision (u = 2^-24), n = 2^10 .. 2^20.  The figure itself is
a placeholder; the text fixes these facts, which pin oracle.alpha_formulas:
  * FFT-based convolution: alpha negative ("not even one bit") for n >= 2^10;
  * original Ozaki scheme: only 2 bits at n = 2^20;
  * single-modulus NTT: slightly larger than the original Ozaki scheme, modest;
  * two-modulus NTT + CRT: 20 bits at n = 2^20, substantially larger.
The CRT column must also equal the alpha the method uses at L = 1 (orc_alpha)."""
import oracle as O


def test_fig1_alpha_table():
    rows = {k: O.alpha_formulas(1 << k) for k in range(10, 21)}
    for k, r in rows.items():
        assert r["fft"] < 0, (k, r)
        assert r["ntt"] >= r["ozaki"] and r["ntt"] - r["ozaki"] <= 4, (k, r)
        assert r["crt"] > r["ntt"] + 5, (k, r)
        assert r["crt"] == O.alpha(1 << k, 1)
    assert rows[20]["ozaki"] == 2
    assert rows[20]["crt"] == 20
    # monotone in n
    for k in range(10, 20):
        for f in ("ozaki", "ntt", "crt"):
            assert rows[k + 1][f] <= rows[k][f]
