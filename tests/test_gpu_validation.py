"""A1's validation rules (include/saga.h "Validation rules"; AEG Def. P:526-534) on the
GPU path: one invalid trace per rule, each rejected with SAGA_ERR_TRACE and the rule's message,
and rejected by the oracle as well (its own rule numbering)."""
import numpy as np
import pytest

from gen import default_place_cfg, make_c1

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_00528_b200 import saga  # noqa: E402
from oracle import oracle as O  # noqa: E402

O.build()


def _mut(field, fn):
    def f():
        d = make_c1()
        a = getattr(d, field).copy()
        fn(a, d)
        setattr(d, field, a)
        return d
    return f


def _swap(a, d):
    a[5], a[6] = a[6], a[5]


def _first_zero(a, d):
    a[1] = a[0]          # call 0 gets no range (CSR not strictly increasing)


def _cttl(d):
    d.call_ttl_base_us = np.full(d.n_calls, 10 ** 6, np.int64)
    d.call_ttl_base_us[3] = 2 * 10 ** 9
    return d


RULES = [
    ("order", _mut("call_t_us", _swap), "strictly increasing in (t, session)"),
    ("time", _mut("call_t_us", lambda a, d: a.__setitem__(0, -5)), "call time outside"),
    ("session_id", _mut("call_session", lambda a, d: a.__setitem__(-1, 99)), "session or AEG node out of range"),
    ("aeg_node", _mut("call_aeg_node", lambda a, d: a.__setitem__(2, 77)), "session or AEG node out of range"),
    ("prompt0", _mut("call_prompt_tokens", lambda a, d: a.__setitem__(4, 0)), "prompt >= 1"),
    ("new_gt_prompt", _mut("call_new_tokens", lambda a, d: a.__setitem__(4, 10 ** 6)), "prompt >= 1"),
    ("work", _mut("call_output_tokens", lambda a, d: a.__setitem__(7, 2 ** 31)), "call work"),
    ("csr", _mut("call_range_off", _first_zero), "call_range_off"),
    ("range_empty", _mut("range_len", lambda a, d: a.__setitem__(3, 0)), "range empty"),
    ("range_outside", _mut("range_block_lo", lambda a, d: a.__setitem__(1, 40)), "range empty, out of bounds, or outside"),
    ("type", _mut("session_type", lambda a, d: a.__setitem__(2, 5)), "session_type >= n_types"),
    ("span", _mut("session_block_len", lambda a, d: a.__setitem__(7, 10 ** 6)), "span outside"),
    ("overlap", _mut("type_shared_len", lambda a, d: a.__setitem__(0, 5)), "overlap"),   # prefix span over session 0's
    ("edge_dst", _mut("edge_dst", lambda a, d: a.__setitem__(0, 999)), "AEG CSR or edge endpoint"),
    ("prob", _mut("edge_p", lambda a, d: a.__setitem__(0, 1.5)), "edge probability"),
    ("ttl", _mut("node_ttl_base_us", lambda a, d: a.__setitem__(0, 2 * 10 ** 9)), "node_ttl_base_us"),
    ("call_ttl", lambda: _cttl(make_c1()), "node_ttl_base_us"),
]


@pytest.mark.parametrize("name,build,msg", RULES, ids=[r[0] for r in RULES])
def test_rule_rejected_on_both_sides(name, build, msg):
    d = build()
    with pytest.raises(ValueError):
        O.Oracle(d, default_place_cfg())
    with pytest.raises(saga.SagaError) as ex:
        saga.Trace(d, default_place_cfg())
    assert ex.value.status == 2, (name, str(ex.value))
    assert msg in str(ex.value), (name, str(ex.value))


def test_valid_c1_accepted():
    saga.Trace(make_c1(), default_place_cfg()).free()
