"""Decoder MLP, Eq. 14: MLP(G(x | Phi_E) | Phi_M) = Theta_hat(x).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

"The MLP we used ... contains 3 linear layers of width 64. Each layer with
ReLU activation, except for the last layer with our custom mapping functions"
(P:302).  Reading C-A5: "a x W" = a affine layers including the output layer,
hidden width W, biases on.  C-O7 forward, C-O14 reverse mode (ReLU'(0) := 0).
Plain float64 matrix products (numpy), no fusion or reordering.
"""
import numpy as np


def forward(layers, z):
    """layers: list of (W [out, in], b [out]); z: [in, n].
    Returns (out [4K, n], pre-activations list, inputs-to-each-layer list)."""
    h = z
    inputs, pres = [], []
    for k, (w, b) in enumerate(layers):
        inputs.append(h)
        a = w @ h + b[:, None]
        pres.append(a)
        h = np.maximum(a, 0.0) if k < len(layers) - 1 else a
    return h, pres, inputs


def backward(layers, pres, inputs, dout):
    """Reverse mode of forward() (C-O14):
      delta_n = dout;  dW_k = delta_k h_{k-1}^T;  db_k = sum_n delta_k;
      delta_{k-1} = (W_k^T delta_k) * [pre_{k-1} > 0];  dz = W_1^T delta_1.
    Returns (list of (dW, db), dz)."""
    grads = [None] * len(layers)
    delta = dout
    for k in range(len(layers) - 1, -1, -1):
        w, _ = layers[k]
        grads[k] = (delta @ inputs[k].T, delta.sum(axis=1))
        dprev = w.T @ delta
        if k > 0:
            dprev = dprev * (pres[k - 1] > 0.0)
        delta = dprev
    return grads, delta
