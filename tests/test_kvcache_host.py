"""Paged KV-cache manager, host logic (dry manager, no GPU): slot assignment,
page reuse, all-or-nothing allocation, block tables, error taxonomy."""
import numpy as np
import pytest

from paper_2605_21603_b200 import opflow as of


def test_slots_fill_pages_in_order_and_positions_continue():
    kv = of.KvCache(layers=1, pages=6, kv_heads=2, dry=True)
    s, p = kv.append([1], [20])
    assert list(p) == list(range(20))
    pages = s // 16
    assert list(s % 16) == [i % 16 for i in range(20)]
    assert len(set(pages[:16])) == 1 and len(set(pages[16:])) == 1 and pages[0] != pages[16]
    s2, p2 = kv.append([1], [5])  # continues the partially filled page
    assert list(p2) == [20, 21, 22, 23, 24]
    assert all(x // 16 == pages[16] for x in s2)
    assert kv.stats() == {"free_pages": 4, "sequences": 1}


def test_release_returns_pages_and_reuse():
    kv = of.KvCache(layers=1, pages=4, kv_heads=1, dry=True)
    a, _ = kv.append([10, 11], [32, 16])  # 2 + 1 pages
    assert kv.stats()["free_pages"] == 1
    kv.release(10)
    assert kv.stats() == {"free_pages": 3, "sequences": 1}
    b, _ = kv.append([12], [48])
    assert set((b // 16).tolist()) <= set(range(4)) and kv.stats()["free_pages"] == 0
    # the live sequence's page was never handed out again
    assert (a[32:] // 16)[0] not in set((b // 16).tolist())


def test_out_of_pages_is_all_or_nothing():
    kv = of.KvCache(layers=1, pages=3, kv_heads=1, dry=True)
    kv.append([1], [16])
    with pytest.raises(of.Error) as e:
        kv.append([2, 3], [16, 17])  # needs 3 pages, 2 free
    assert e.value.code == of.ERRC.index("ConfigError") and "out of pages" in str(e.value)
    assert kv.stats() == {"free_pages": 2, "sequences": 1}


def test_duplicate_ids_in_one_call_append_in_order():
    kv = of.KvCache(layers=1, pages=4, kv_heads=1, dry=True)
    s, p = kv.append([5, 5], [10, 10])
    assert list(p) == list(range(20))
    tab, lens = kv.block_table([5], 4)
    assert lens.tolist() == [20] and tab[0, 2] == -1
    assert (s[:16] // 16 == tab[0, 0]).all() and (s[16:] // 16 == tab[0, 1]).all()


def test_block_table_errors():
    kv = of.KvCache(layers=1, pages=8, kv_heads=1, dry=True)
    kv.append([1], [40])
    with pytest.raises(of.Error) as e:
        kv.block_table([1], 2)  # spans 3 pages
    assert e.value.code == of.ERRC.index("ShapeMismatch")
    with pytest.raises(of.Error) as e:
        kv.block_table([99], 4)
    assert e.value.code == of.ERRC.index("UnknownTensor")
    with pytest.raises(of.Error):
        of.KvCache(layers=1, pages=8, kv_heads=1, kv_layout=2, dry=True)
