"""Cordeau instance files and solution files against the
reference's own parse_instance / write_solution / read_solution results
(tests/golden/formats/, made by make_formats_golden.py)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2605_05208_b200.formats import ParseError, parse_instance, read_solution, write_solution
from paper_2605_05208_b200.model import Route, Solution

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")
MAN = json.load(open(os.path.join(HERE, "manifest.json")))


@pytest.mark.parametrize("key", sorted(MAN["cases"]))
def test_parse_instance_equals_reference(key):
    fname, variant, relax = key.split("|")
    want = MAN["cases"][key]
    inst = parse_instance(os.path.join(HERE, fname), variant, relax_fleet=relax == "1")
    assert hashlib.sha256(np.ascontiguousarray(inst.dist).tobytes()).hexdigest() == want["dist_sha"]
    assert list(map(int, inst.labels)) == want["labels"]
    assert inst.name == want["name"] and inst.n_depots == want["n_depots"]
    assert (float(inst.fleet_per_depot), float(inst.capacity), float(inst.max_duration)) == \
        (want["fleet"], want["capacity"], want["max_duration"])


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(MAN["cases"]))
def test_solution_file_equals_reference(key, tmp_path):
    """write_solution (route distances and loads from the device simulation) is byte-identical."""
    fname, variant, relax = key.split("|")
    want = MAN["cases"][key]
    inst = parse_instance(os.path.join(HERE, fname), variant, relax_fleet=relax == "1")
    sol = Solution([Route(d, a, list(c)) for d, a, c in want["routes"]])
    out = tmp_path / "s.sol"
    write_solution(sol, out, inst)
    assert out.read_text() == open(os.path.join(HERE, want["sol_file"])).read()


@pytest.mark.parametrize("key", sorted(MAN["cases"]))
def test_read_solution_equals_reference(key):
    fname, variant, relax = key.split("|")
    want = MAN["cases"][key]
    inst = parse_instance(os.path.join(HERE, fname), variant, relax_fleet=relax == "1")
    back = read_solution(os.path.join(HERE, want["sol_file"]), inst)
    assert [[r.depart, r.arrive, r.customers] for r in back.routes] == [list(x) for x in want["read_back"]]


@pytest.mark.parametrize("fname", sorted(MAN["errors"]))
def test_parse_errors_equal_reference(fname):
    variant, msg = MAN["errors"][fname]
    with pytest.raises(ParseError) as ei:
        parse_instance(os.path.join(HERE, fname), variant)
    assert str(ei.value).replace(HERE + "/", "") == msg
