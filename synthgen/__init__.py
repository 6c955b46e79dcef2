"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no layer maths, no scheduling).
It only:
  * lists each model's parameters (name, shape, init kind)   -> manifest.py
  * draws seeded random weights / inputs with numpy PCG64     -> gen.py
  * encodes them as bf16 bit patterns and writes weight files -> gen.py

Recipe: SURVEY.md §8(c) C1.3 (seeds, distributions), C1.2 (model list).
"""
from .manifest import MODELS, MODEL_INDEX, manifest, input_shape
from .gen import (weights, weight_file, image_batch, mnist_batch, bert_ids,
                  model_input, f32_to_bf16_bits, bf16_bits_to_f32, pad_channels)

__all__ = ["MODELS", "MODEL_INDEX", "manifest", "input_shape", "weights",
           "weight_file", "image_batch", "mnist_batch", "bert_ids", "model_input",
           "f32_to_bf16_bits", "bf16_bits_to_f32", "pad_channels"]
