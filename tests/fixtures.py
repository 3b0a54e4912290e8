"""Shared test fixtures: golden cases as coldgen objects (no method arithmetic here)."""
import json
import os

import numpy as np

import coldgen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


_SIDES = {"user": coldgen.USER, "ad": coldgen.AD, "cross": coldgen.CROSS}


def worked_example(head="one", linear_log=True):
    """SURVEY P-4 worked example (tests/golden/p4_worked_example.json). Parameters are kept
    in fp64 (0.3 etc. are not fp32 values); tables are exact in fp32."""
    gd = load_golden("p4_worked_example.json")
    groups = []
    for g in gd["groups"]:
        groups.append(coldgen.Group(g["name"], _SIDES[g["side"]], g["card"],
                                    tuple(g["bag"]) if "bag" in g else None,
                                    g.get("user_ref", -1), g.get("ad_ref", -1)))
    h = gd["one_wide_head"] if head == "one" else gd["two_wide_head"]
    width_last = len(h["W2"])
    schema = coldgen.Schema("P4", tuple(groups), gd["k"], (2, width_last), linear_log)
    params = coldgen.Params(
        tables=[np.asarray(t, np.float32) for t in gd["tables"]], table_dtype="f32",
        se_w=np.asarray(gd["se_w"], np.float64), se_b=np.asarray(gd["se_b"], np.float64),
        fc_w=[np.asarray(gd["W1"], np.float64), np.asarray(h["W2"], np.float64)],
        fc_b=[np.asarray(gd["b1"], np.float64), np.asarray(h["b2"], np.float64)],
        precision="f32", init="golden", seed=0)
    ads = gd["ads"]
    batch = coldgen.Batch(
        R=1, ad_offsets=np.asarray([0, len(ads)], np.int32),
        ids=[np.asarray(gd["user_bag"], np.int32), np.asarray(ads, np.int32), None],
        offs=[np.asarray([0, len(gd["user_bag"])], np.int32), None, None],
        bids=None, req_ids=np.asarray([0]))
    return schema, params, batch, gd["expected"]


def small_case(schema_name="tiny", R=3, n_ads=(5, 17, 1), precision="f32", seed=7, cap=None,
               dist="uniform", init="xavier", se="random", bids=False):
    """Small seeded case over a (possibly cardinality-capped) schema."""
    sch = {"tiny": coldgen.schema_tiny, "paper": coldgen.schema_paper, "full": coldgen.schema_full}[schema_name]()
    if cap is not None:
        sch = coldgen.scaled_schema(sch, cap)
    params = coldgen.make_params(sch, seed=seed, precision=precision, init=init, se=se)
    batch = coldgen.make_batch(sch, R, list(n_ads) if not isinstance(n_ads, int) else n_ads,
                               seed=seed + 1, dist=dist, bids=bids)
    return sch, params, batch


def bag_schema():
    """A schema exercising ad bags (ragged, possibly empty) and bag x bag crosses."""
    g = [
        coldgen.Group("u_single", coldgen.USER, 37),
        coldgen.Group("u_bag", coldgen.USER, 53, (0, 5)),
        coldgen.Group("a_single", coldgen.AD, 41),
        coldgen.Group("a_bag", coldgen.AD, 29, (0, 4)),
    ]
    g.append(coldgen.Group("ubag_x_abag", coldgen.CROSS, 97, None, 1, 3))
    g.append(coldgen.Group("usingle_x_asingle", coldgen.CROSS, 61, None, 0, 2))
    g.append(coldgen.Group("ubag_x_asingle", coldgen.CROSS, 1, None, 1, 2))
    return coldgen.Schema("bags", tuple(g), 4, (16, 8, 2), True)
