"""Exponentially windowed Fourier pipeline (mirror of reference ``transform.py``).

* ``eta_from_kappa``, ``frequency_grid``, ``TimeSignal`` and ``forward_mft``
  are per-run host setup ("forward_mft is host-side setup,
  O(N log N) per signal") and keep the reference's numpy formulas.
* The time reconstruction — ``conjugate_fill`` + window + inverse DFT x N +
  imaginary-residue check + e^{eta n dt} rescale (``transform.py:137-203``)
  — runs on the GPU for any number of DOF columns at once
  (``ewb_window_idft``).  ``inverse_mft(spectrum, window, eta)`` keeps the
  reference signature.
"""

from __future__ import annotations

import logging
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

WINDOW_KINDS = ("rectangular", "hanning", "blackman")
WINDOW_CODE = {"rectangular": 0, "hanning": 1, "blackman": 2}
IMAG_RESIDUE_CHECK = 1e-10
IMAG_RESIDUE_HARD_ERROR = 1e-8

log = logging.getLogger(__name__)


class SpectrumSymmetryError(RuntimeError):
    """Inverse transform produced a significantly complex signal."""


@dataclass(frozen=True)
class TimeSignal:
    kind: str = "zero"
    amplitude: float = 0.0
    times: np.ndarray | None = field(default=None)
    values: np.ndarray | None = field(default=None)

    def sample(self, period: float, n_samples: int) -> np.ndarray:
        t = np.arange(n_samples) * (period / n_samples)
        if self.kind == "zero":
            return np.zeros(n_samples)
        if self.kind == "heaviside":
            return np.full(n_samples, float(self.amplitude))
        if self.kind == "tabulated":
            if self.times is None or self.values is None:
                raise ValueError("tabulated signal without samples")
            return np.interp(t, self.times, self.values)
        raise ValueError(f"unknown signal kind {self.kind!r}")

    @classmethod
    def heaviside(cls, amplitude: float) -> "TimeSignal":
        return cls(kind="heaviside", amplitude=float(amplitude))

    @classmethod
    def zero(cls) -> "TimeSignal":
        return cls(kind="zero")

    @classmethod
    def tabulated(cls, times, values) -> "TimeSignal":
        times = np.asarray(times, dtype=float)
        values = np.asarray(values, dtype=float)
        if times.ndim != 1 or times.shape != values.shape or times.size < 2:
            raise ValueError("tabulated signal needs matching 1-D arrays")
        if not np.all(np.diff(times) > 0):
            raise ValueError("tabulated signal times must be increasing")
        return cls(kind="tabulated", times=times, values=values)


@dataclass
class Spectrum:
    values: np.ndarray
    period: float
    eta: float

    @property
    def n_omega(self) -> int:
        return len(self.values)

    @property
    def delta_omega(self) -> float:
        return 2.0 * math.pi / self.period

    def frequencies(self) -> np.ndarray:
        return np.arange(self.n_omega) * self.delta_omega - 1j * self.eta


def eta_from_kappa(kappa: float, period: float) -> float:
    if kappa < 0:
        raise ValueError("kappa must be >= 0")
    if period <= 0:
        raise ValueError("period must be positive")
    return kappa * math.log(10.0) / period


def frequency_grid(period: float, n_omega: int, eta: float) -> np.ndarray:
    if n_omega % 2 or n_omega < 4:
        raise ValueError("n_omega must be even and >= 4")
    dw = 2.0 * math.pi / period
    return np.arange(n_omega // 2 + 1) * dw - 1j * eta


def forward_mft(signal: TimeSignal, period: float, n_omega: int, eta: float) -> Spectrum:
    if n_omega < 2:
        raise ValueError("need at least 2 samples")
    x = signal.sample(period, n_omega)
    dt = period / n_omega
    return Spectrum(values=np.fft.fft(x * np.exp(-eta * dt * np.arange(n_omega))) / n_omega,
                    period=period, eta=eta)


def forward_mft_batch(signals, period: float, n_omega: int, eta: float,
                      n_keep: int | None = None) -> np.ndarray:
    """forward_mft of many signals at once: (len(signals), n_keep) complex,
    the first n_keep (default all n_omega) frequencies of each spectrum.

    Heaviside signals are constant, H(0) = 1 (transform.py:65-66), so their
    spectra are amplitude x the spectrum of the damped unit step (linearity;
    equal to the per-signal FFT to 1 ulp).  Tabulated signals go through one
    batched FFT.  cfg2 has 15,361 signals: per-signal transforms cost ~0.6 s
    of setup, this ~10 ms."""
    if n_omega < 2:
        raise ValueError("need at least 2 samples")
    dt = period / n_omega
    damp = np.exp(-eta * dt * np.arange(n_omega))
    nk = n_omega if n_keep is None else int(n_keep)
    amp = np.zeros(len(signals))
    tab = []
    for i, sig in enumerate(signals):
        if sig.kind == "heaviside":
            amp[i] = float(sig.amplitude)
        elif sig.kind != "zero":
            tab.append(i)
    out = amp[:, None] * (np.fft.fft(damp) / n_omega)[None, :nk]
    if tab:
        x = np.stack([signals[i].sample(period, n_omega) for i in tab])
        out[tab] = (np.fft.fft(x * damp, axis=1) / n_omega)[:, :nk]
    return out


def conjugate_fill(half_values, period: float, eta: float) -> Spectrum:
    """Host bookkeeping for API parity; the device path fuses this step."""
    half = np.asarray(half_values, dtype=complex)
    if half.ndim != 1 or half.size < 2:
        raise ValueError("half spectrum must be 1-D with at least 2 values")
    nh = half.size
    n = 2 * (nh - 1)
    full = np.empty(n, dtype=complex)
    full[:nh] = half
    full[0] = half[0].real
    full[nh - 1] = half[nh - 1].real
    full[nh:] = np.conj(full[1:n - nh + 1][::-1])
    return Spectrum(values=full, period=period, eta=eta)


def window_weights(kind: str, n_omega: int) -> np.ndarray:
    if n_omega < 2:
        raise ValueError("need at least 2 samples")
    if kind == "rectangular":
        return np.ones(n_omega)
    ph = 2.0 * math.pi * np.arange(n_omega) / n_omega
    if kind == "hanning":
        return 0.5 * (1.0 + np.cos(ph))
    if kind == "blackman":
        return 0.42 + 0.5 * np.cos(ph) + 0.08 * np.cos(2.0 * ph)
    raise ValueError(f"unknown window kind {kind!r}; expected one of {WINDOW_KINDS}")


def windowed_inverse_device(half_dev, window: str, eta: float, period: float):
    """GPU reconstruction of D columns: half_dev (n_half, D) complex128 cuda.

    Returns (series (N, D) float64 cuda, residue (D,) float64 cuda).
    """
    import torch

    lib = _lib.require_cuda()
    if window not in WINDOW_CODE:
        raise ValueError(f"unknown window kind {window!r}; expected one of {WINDOW_KINDS}")
    half_dev = half_dev.contiguous()
    nh, D = half_dev.shape
    N = 2 * (nh - 1)
    out = torch.empty((N, D), dtype=torch.float64, device=half_dev.device)
    res = torch.empty((D,), dtype=torch.float64, device=half_dev.device)
    _lib.check(lib.ewb_window_idft(_lib.ptr(half_dev), nh, D, WINDOW_CODE[window], float(eta),
                                   float(period), _lib.ptr(out), _lib.ptr(res),
                                   _lib.stream_handle()), "ewb_window_idft")
    return out, res


def check_residue(residue: float) -> None:
    """transform.py:189-200: raise above 1e-8, warn above 1e-10."""
    if residue > IMAG_RESIDUE_HARD_ERROR:
        raise SpectrumSymmetryError(
            f"imaginary residue {residue:.3e} exceeds {IMAG_RESIDUE_HARD_ERROR}; "
            "spectrum is not conjugate symmetric")
    if residue > IMAG_RESIDUE_CHECK:
        log.warning("inverse transform imaginary residue %.3e above %.0e",
                    residue, IMAG_RESIDUE_CHECK)


def inverse_mft(spectrum: Spectrum, window: str, eta: float) -> np.ndarray:
    """Reference signature (``transform.py:179``) on the device.

    The device kernel rebuilds the full spectrum from bins 0..N/2; a
    spectrum that is not conjugate symmetric is detected on the host first
    (the reference would see it as a large imaginary residue).
    """
    import torch

    vals = np.asarray(spectrum.values, dtype=complex)
    n = len(vals)
    if n % 2:
        raise ValueError("device inverse needs an even number of bins")
    nh = n // 2 + 1
    mirror = np.conj(vals[1:nh - 1][::-1])
    scale = max(np.abs(vals).max(), 1e-300)
    if np.abs(vals[nh:] - mirror).max() > 1e-8 * scale or \
            abs(vals[0].imag) > 1e-8 * scale or abs(vals[nh - 1].imag) > 1e-8 * scale:
        raise SpectrumSymmetryError("spectrum is not conjugate symmetric")
    half = torch.from_numpy(np.ascontiguousarray(vals[:nh]).reshape(nh, 1)).cuda()
    out, res = windowed_inverse_device(half, window, eta, spectrum.period)
    check_residue(float(res[0]))
    return out[:, 0].cpu().numpy()
