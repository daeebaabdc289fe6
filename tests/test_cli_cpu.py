"""cli.run_cli argument handling that never reaches the GPU (usage errors, exit code 2),
mirroring reference tests/test_cli.py:53-70."""

from paper_2305_09493_b200.cli import run_cli


def test_missing_input_is_usage_error(capsys):
    assert run_cli([]) == 2
    assert "an input file is required" in capsys.readouterr().err


def test_missing_file_is_usage_error(tmp_path, capsys):
    assert run_cli([str(tmp_path / "nope.spv")]) == 2
    assert "no such file" in capsys.readouterr().err


def test_both_input_forms_rejected(tmp_path, capsys):
    f = tmp_path / "a.spv"
    f.write_bytes(b"")
    assert run_cli([str(f), "-d", str(f)]) == 2


def test_stdin_only_for_text_tool(capsys):
    assert run_cli(["-"]) == 2
    assert run_cli(["--tool", "val", "-"]) == 2


def test_batch_missing_file_and_output_conflict(tmp_path, capsys):
    f = tmp_path / "a.spv"
    f.write_bytes(b"")
    assert run_cli([str(f), str(tmp_path / "b.spv"), "--out-dir", str(tmp_path / "o")]) == 2
    assert run_cli([str(f), str(f), "-o", str(tmp_path / "x")]) == 2
