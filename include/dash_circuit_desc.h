/*
 * Plain-data description of a quantized Dash circuit, shared by the product
 * library (libdashgpu), the CPU oracle (oracle/liboracle) and the reference
 * harness (oracle/_ref/libdashref).  It is the C-ABI image of
 * dash::Circuit / dash::Layer (reference: proj/core/include/dash/circuit.hpp:13-19,
 * proj/core/include/dash/layer.hpp:16-54): a chain of layers over a CRT base of
 * k primes, weights row-major [out][in] (Dense) or [out_ch][in_ch][f][f]
 * (Conv2d, square filters, no padding).
 *
 * Extensions beyond the reference (parity is pinned
 * by the C restatement only, the reference has no such layers -- SURVEY.md
 * section 8(d) "ResNet-20 extension notes"):
 *   DASH_LAYER_PAD2D  zero padding of a [C][H][W] tensor by `pad` cells on
 *                     every side; pad cells hold the zero-wire label
 *                     (garble.cpp:157: zero wire i = prf.label(i, p_i)), so
 *                     an unmodified Conv2d after it is a padded convolution.
 *   DASH_LAYER_ADD    lane-wise label sum of two equal-shape tensors (the
 *                     residual add; free, like the reference's free_add,
 *                     gadgets.hpp:108-118).
 *   src / src2        DAG inputs: 0 = previous layer's output (the
 *                     reference's chain), j + 1 = output of layer j, -1 = the
 *                     circuit input.  src2 is the second operand of ADD.
 * Layers without extensions keep src = src2 = pad = 0 and serialize exactly
 * as the reference does.
 */
#ifndef DASH_CIRCUIT_DESC_H
#define DASH_CIRCUIT_DESC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dash::LayerKind (layer.hpp:16-22) */
enum {
    DASH_LAYER_DENSE = 1,
    DASH_LAYER_CONV2D = 2,
    DASH_LAYER_RELU = 3,
    DASH_LAYER_SIGNACT = 4,
    DASH_LAYER_FLATTEN = 5,
    DASH_LAYER_PAD2D = 6, /* extension */
    DASH_LAYER_ADD = 7    /* extension */
};

typedef struct dash_layer_desc {
    int32_t kind;            /* DASH_LAYER_* */
    int32_t private_weights; /* projection-gate linear layer (layer.hpp:27) */
    uint32_t in_dim, out_dim;                 /* Dense */
    uint32_t in_ch, out_ch, filter, stride;   /* Conv2d */
    const int64_t* q_weights; /* weight_count() entries, or NULL */
    uint64_t n_weights;
    const int64_t* q_biases;  /* bias_count() entries, or NULL (= all zero) */
    uint64_t n_biases;
    int32_t src, src2;        /* extension: DAG inputs (see above) */
    uint32_t pad;             /* extension: PAD2D cells per side */
} dash_layer_desc;

typedef struct dash_circuit_desc {
    int32_t k;                /* CRT base size, 1..16 */
    uint32_t rank;            /* input rank, 1..8 */
    uint32_t input_shape[8];
    double sign_target;       /* 1.0 = full-accuracy sign spec */
    double alpha;             /* quant.alpha (carried into the gc header) */
    uint32_t n_layers;
    const dash_layer_desc* layers;
} dash_circuit_desc;

#ifdef __cplusplus
}
#endif

#endif
