"""Pins for the oracle's a1 classifier `orc_classify` with its DEFAULT thresholds (R13), taken
directly from SPEC.md's classifier examples -- not from the calibration module.

R13 represents the smart classifier as per-modality footprint thresholds (thr_mc, thr_ct):
class M if f < thr_mc[mod], else C if f < thr_ct[mod], else T.
  naive: text (inf, inf), image (0, inf), video (0, 0)
  smart default:                         text (4096, inf), image (0, inf), video (0, 8192)
"""
import numpy as np
import pytest

import oracle as O
import tracegen as T

M, C, TR = 0, 1, 2
TEXT, IMAGE, VIDEO = 0, 1, 2
NAIVE = O.model(thresholds=O.NAIVE_THR)


@pytest.mark.parametrize("f", [1, 10, 200, 4095, 4096, 9000, 10_000, 131_072])
def test_naive_text_any_size_is_motorcycle(f):
    # SPEC.md:312 "Text, any size -> Motorcycle" ("text -> motorcycles")
    assert O.classify(TEXT, f, NAIVE) == M


@pytest.mark.parametrize("f", [1, 729, 793, 1241])
def test_naive_image_is_car(f):
    # SPEC.md:313 "Image -> Car"
    assert O.classify(IMAGE, f, NAIVE) == C


def test_naive_8_frame_video_is_truck():
    # SPEC.md:314 "Video, 8-frame clip -> Truck (even though its footprint overlaps images)":
    # 8 frames x 196 tokens + a 50-token prompt = 1,618 tokens, inside the image range of Fig. 2a
    f = 8 * 196 + 50
    assert O.classify(VIDEO, f, NAIVE) == TR
    assert O.classify(IMAGE, f, NAIVE) == C                  # same footprint as an image: still Car


def test_smart_9000_token_text_is_car():
    # SPEC.md:333 / :470 / :614 "a 9,000-token text prompt ... -> Car"
    assert O.classify(TEXT, 9000) == C


def test_smart_800_token_video_is_car():
    # SPEC.md:334 / :614 "an 800-token video clip -> Car, not Truck"
    assert O.classify(VIDEO, 800) == C


def test_smart_long_video_is_truck_and_boundaries():
    # R13 smart thresholds: video T from 8,192 tokens; text C from 4,096 tokens; images never T
    assert O.classify(VIDEO, 8191) == C and O.classify(VIDEO, 8192) == TR
    assert O.classify(VIDEO, 512 * 196 + 50) == TR           # the longest generated clip
    assert O.classify(TEXT, 4095) == M and O.classify(TEXT, 4096) == C
    assert O.classify(TEXT, 0xFFFFFFFE) == C                  # text never becomes a truck
    assert all(O.classify(IMAGE, f) == C for f in (1, 729, 4096, 65536))


def test_smart_typical_text_is_motorcycle_95pct():
    # SPEC.md:323 / :614 "text-typical points land in the Motorcycle cluster for >= 95% of text
    # samples" -- on the default text profile of the generator (LN(200, 1.0) in
    # [10, 1e4]); analytically P(f >= 4096) = P(Z > ln(4096/200)) ~ 0.13 %.
    tr = T.generate(np.array([T.make_replica(11, r, 2000, 2.0, (1.0, 0.0, 0.0)) for r in range(4)]))
    cls = np.array([O.classify(int(m), int(f)) for m, f in zip(tr.modality, tr.footprint)])
    assert np.all(tr.modality == TEXT)
    assert (cls == M).mean() >= 0.95


def test_simulation_uses_the_classifier():
    # SPEC.md:470 "tcm + 9,000-token text -> class Car": the engine records the class at ingest
    tr = T.from_requests([[0, 9000, 0, 1, TEXT], [5, 800, 100_000, 1, VIDEO], [9, 200, 0, 1, TEXT],
                          [12, 20_000, 1_000_000, 1, VIDEO]])
    r = O.simulate(tr.arrival_us, tr.footprint, tr.inline_us, tr.out_tokens, tr.modality, policy=O.TCM,
                   kv_capacity=65536)
    assert r.cls.tolist() == [C, C, M, TR]
