"""CPU: the graph descriptions committed for the reference arm
(oracle/fixtures/*.json) are exactly what the product's builders emit, and
the reference's own build_graph accepts them (same topological order)."""
import json

import pytest

from oracle.fixtures import make_fixtures


@pytest.mark.usefixtures("built")
def test_fixtures_match_builders():
    for name, text in make_fixtures.expected().items():
        assert json.loads(make_fixtures.load(name)) == json.loads(text), name


def test_fixtures_build_in_reference(ref):
    from paper_2605_21603_b200 import opflow as of
    for name in make_fixtures.expected():
        desc = make_fixtures.load(name)
        g_ref, _ = ref.graph_and_plan(desc)
        ours = json.loads(of.build_graph(desc).dump_json)
        assert [o["name"] for o in json.loads(g_ref)["ops"]] == [o["name"] for o in ours["ops"]], name
